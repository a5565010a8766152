"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list.

    python tools/launch_summary.py launches.csv
Prints, per kernel: launches, mean and total device time, share of the total.
(ncu serialises launches and runs them cold: compare shares, not absolutes.)
"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
agg = collections.defaultdict(list)
for r in rows[hi + 1:]:
    try:
        v = float(r[vi].replace(",", ""))
    except (ValueError, IndexError):
        continue
    agg[r[ki].split("(")[0].replace("void ", "")].append(v)
tot = sum(sum(v) for v in agg.values())
print(f"{'kernel':58s} {'n':>5s} {'mean_us':>9s} {'total_us':>10s} {'share':>6s}")
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"{k[:58]:58s} {len(v):5d} {sum(v) / len(v) / 1e3:9.2f} {sum(v) / 1e3:10.1f} {100 * sum(v) / tot:5.1f}%")
print(f"total {tot / 1e3:.1f} us over {sum(len(v) for v in agg.values())} launches")
