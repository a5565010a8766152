#!/usr/bin/env python
"""Achieved HBM bandwidth per kernel from an ncu launch list with DRAM metrics.

    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,\\
        dram__throughput.avg.pct_of_peak_sustained_elapsed --csv --log-file x.csv <cmd>
    python tools/hbm_summary.py x.csv
Per kernel: launches, median duration, median DRAM bytes (read + write) and
their ratio (cold, serialised launches).
"""
import collections
import csv
import statistics
import sys

UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
TIME = {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "nsecond": 1e-9}

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ki, mi, vi, ui, idx = (h.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value",
                                             "Metric Unit", "ID"))
launch = collections.defaultdict(dict)
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    launch[(r[idx], r[ki].split("(")[0])][r[mi]] = (float(r[vi].replace(",", "")), r[ui])
per = collections.defaultdict(list)
for (_, name), m in launch.items():
    per[name].append(m)
print(f"{'kernel':28s} {'n':>4s} {'median':>10s} {'DRAM bytes':>12s} {'GB/s':>8s} {'% peak':>7s}")
for name, ms in per.items():
    t = statistics.median(m["gpu__time_duration.sum"][0] * TIME[m["gpu__time_duration.sum"][1]]
                          for m in ms)
    b = statistics.median(sum(m[k][0] * UNITS[m[k][1]] for k in ("dram__bytes_read.sum",
                                                                    "dram__bytes_write.sum"))
                          for m in ms)
    pct = statistics.median(m["dram__throughput.avg.pct_of_peak_sustained_elapsed"][0] for m in ms)
    print(f"{name:28s} {len(ms):4d} {t * 1e6:8.1f}us {b / 1e6:10.2f}MB {b / t / 1e9:8.0f} {pct:6.1f}%")
