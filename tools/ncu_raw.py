#!/usr/bin/env python
"""Key raw metrics of one kernel in an ncu --set full report, as JSON.

    python tools/ncu_raw.py report.ncu-rep > raw.json
"""
import csv
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active"]


def main(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, units, v = rows[0], rows[1], rows[2]
    res = {"Kernel Name": v[h.index("Kernel Name")]}
    for k in KEYS:
        if k in h:
            i = h.index(k)
            res[k] = v[i]
            res[k + " [unit]"] = units[i]
    stalls = {}
    for i, k in enumerate(h):
        if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("_not_issued"):
            try:
                stalls[k.replace("smsp__pcsamp_warps_issue_stalled_", "")] = float(v[i].replace(",", ""))
            except ValueError:
                pass
    tot = sum(stalls.values()) or 1.0
    res["stall_shares"] = {k: round(x / tot, 4) for k, x in sorted(stalls.items(), key=lambda kv: -kv[1]) if x > 0}
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main(sys.argv[1])
