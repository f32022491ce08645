"""Record the DRAM traffic of the repeated-addition kernel from an ncu launch list.

  python tools/traffic_from_launches.py <launches.csv> <config-key> <n> <elem-bytes> [--copy-to DIR]

<launches.csv> is the CSV of
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
      --clock-control none --csv --log-file <csv> python tools/profile_one.py ...
The repeated-addition launches (k_bform, k_aform, k_bgroup) of the (single)
product in the list are summed
(a Case A row split runs both); the bytes go to profiles/ncu_traffic.json[<config-key>] (bench.py reports them as
roofline.traffic next to the algorithmic bytes 3 n^2 x elem: X and Y read
once, Z written once).
"""
import csv
import json
import os
import shutil
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    path, key, n, es = sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4])
    copy_to = sys.argv[sys.argv.index("--copy-to") + 1] if "--copy-to" in sys.argv else None
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, mi, vi, ii, ui = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value",
                                                  "ID", "Metric Unit"))
    scale = {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1.0,
             "second": 1.0, "nsecond": 1e-9, "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6,
             "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
    launches = {}
    for r in rows[1:]:
        if not any(x in r[ki] for x in ("k_bform", "k_aform", "k_bgroup")):
            continue
        d = launches.setdefault(int(r[ii]), {"kernel": r[ki]})
        d[r[mi]] = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
    if not launches:
        sys.exit(f"no repeated-addition kernel launch in {path}")
    # one product per launch list (tools/profile_one.py --reps 1): a Case A row
    # split launches k_aform and k_bform; both belong to the product
    rd = sum(d["dram__bytes_read.sum"] for d in launches.values())
    wr = sum(d["dram__bytes_write.sum"] for d in launches.values())
    t = sum(d["gpu__time_duration.sum"] for d in launches.values())  # seconds
    last = launches[max(launches)]
    src = path
    if copy_to:
        os.makedirs(os.path.join(ROOT, copy_to), exist_ok=True)
        dst = os.path.join(copy_to, os.path.basename(path))
        shutil.copy(path, os.path.join(ROOT, dst))
        src = dst
    # the kernels that ran (the form not chosen on the device exits at once:
    # named only when it took at least 1% of the product's kernel time)
    kernel = " + ".join(d["kernel"].split("(")[0].replace("void ", "").replace("afmm_dev::", "")
                        .replace("unnamed>::", "") for _, d in sorted(launches.items())
                        if d["gpu__time_duration.sum"] >= 0.01 * t)
    entry = {
        "bytes_per_launch": rd + wr, "dram_read": rd, "dram_write": wr,
        "kernel_time_s": t, "kernel": kernel, "source": src,
        "algorithmic_bytes": 3 * n * n * es,
        "note": "DRAM bytes of one launch (ncu, cold caches); algorithmic = X and Y read once, "
                "Z written once",
    }
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    data = json.load(open(tp)) if os.path.exists(tp) else {}
    data[key] = entry
    with open(tp, "w") as f:
        json.dump(data, f, indent=1)
    print(key, kernel, f"{(rd + wr) / 1e9:.3f} GB per launch, {t * 1e3:.3f} ms")


if __name__ == "__main__":
    main()
