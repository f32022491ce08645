"""Summarise an `ncu --set full` capture of k_bform and record its DRAM traffic.

  python tools/ncu_summary.py <report.ncu-rep> <config-key> [--out profiles/rNN/x.json]

Writes the key metrics (time, dram bytes, pipe utilisation, issue activity,
stall reasons) as JSON and updates profiles/ncu_traffic.json[<config-key>],
which bench.py reports as roofline.traffic.
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

KEYS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread",
    "launch__occupancy_limit_shared_mem",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "lts__t_bytes.sum",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_branch_resolving_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
]

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "ns": 1e-9, "nsecond": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3,
         "s": 1.0, "second": 1.0}


def main():
    rep, key = sys.argv[1], sys.argv[2]
    out = None
    if "--out" in sys.argv:
        out = sys.argv[sys.argv.index("--out") + 1]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    launches = []
    for vals in rows[2:]:
        d = {}
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                v = vals[i].replace(",", "")
                try:
                    f = float(v)
                except ValueError:
                    continue
                u = units[i]
                if u in SCALE:
                    f *= SCALE[u]
                    u = "s" if u in ("ns", "nsecond", "us", "usecond", "ms", "msecond", "s",
                                     "second") else "byte"
                d[k] = {"value": f, "unit": u}
        d["kernel"] = vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
        launches.append(d)
    summary = {"report": os.path.relpath(rep, ROOT), "config": key, "launches": launches}
    if out:
        with open(out, "w") as f:
            json.dump(summary, f, indent=1)
    first = launches[0]
    traffic = first["dram__bytes_read.sum"]["value"] + first["dram__bytes_write.sum"]["value"]
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            table = json.load(f)
    except (OSError, ValueError):
        table = {}
    table[key] = {"bytes_per_launch": traffic,
                  "dram_read": first["dram__bytes_read.sum"]["value"],
                  "dram_write": first["dram__bytes_write.sum"]["value"],
                  "kernel_time_s": first["gpu__time_duration.sum"]["value"],
                  "source": os.path.relpath(rep, ROOT)}
    with open(path, "w") as f:
        json.dump(table, f, indent=1)
    print(json.dumps(table[key], indent=1))


if __name__ == "__main__":
    main()
