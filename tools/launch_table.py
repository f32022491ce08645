"""Per-kernel table of an ncu launch list (dev tool).

  python tools/launch_table.py launches.csv [--last N]

Prints each launch's duration, DRAM bytes and achieved DRAM bandwidth, then
the per-kernel sums over the last N launches (default: all), so the prepass
kernels' share of a product and their distance from HBM bandwidth can be read
at a glance."""
import collections
import csv
import sys


def load(path):
    rows = list(csv.reader(l for l in open(path) if not l.startswith("==")))
    h = rows[0]
    ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    d = collections.OrderedDict()
    for r in rows[1:]:
        d.setdefault(r[0], {"name": r[ki]})[r[mi]] = float(r[vi].replace(",", ""))
    return list(d.values())


def short(name):
    base = name.split("(")[0]
    return base.split("::")[-1][:48]


def main():
    path = sys.argv[1]
    last = int(sys.argv[sys.argv.index("--last") + 1]) if "--last" in sys.argv else 0
    ls = load(path)
    if last:
        ls = ls[-last:]
    tot = collections.OrderedDict()
    for m in ls:
        t = m.get("gpu__time_duration.sum", 0.0)
        b = m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
        print(f"{short(m['name']):48s} {t / 1e3:10.1f} us {b / 1e6:9.1f} MB {b / t if t else 0:7.0f} GB/s")
        e = tot.setdefault(short(m["name"]), [0.0, 0.0, 0])
        e[0] += t
        e[1] += b
        e[2] += 1
    print("-- per kernel")
    for k, (t, b, c) in tot.items():
        print(f"{k:48s} x{c:<3d} {t / 1e3:10.1f} us {b / 1e6:9.1f} MB")


if __name__ == "__main__":
    main()
