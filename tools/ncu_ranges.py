"""Instruction / stall shares of an ncu report grouped by source-line ranges
of the kernel's own file (other files are grouped by file name).

    python tools/ncu_ranges.py report.ncu-rep name:lo-hi [name:lo-hi ...]

Lines outside every range are reported as "other" (needs -lineinfo).  Only
SASS rows are counted (the source rows of --print-source=cuda,sass repeat
their SASS totals).
"""
import csv
import collections
import subprocess
import sys

rep = sys.argv[1]
ranges = []
for a in sys.argv[2:]:
    name, _, span = a.partition(":")
    lo, _, hi = span.partition("-")
    ranges.append((name, int(lo), int(hi)))
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hi = [i for i, x in enumerate(rows) if x and x[0] == "Line No"][0]
h = rows[hi]
iex = h.index("Instructions Executed")
ist = h.index("Warp Stall Sampling (All Samples)")
ins = collections.Counter()
stl = collections.Counter()
cur = None
first_file = None
cur_file = None
for x in rows:
    if len(x) >= 2 and x[0] == "File Path":
        cur_file = x[1]
        first_file = first_file or cur_file
        continue
    if len(x) <= iex or x[0] == "Line No":
        continue
    if x[0]:
        if x[0].isdigit():
            cur = int(x[0])
        continue  # source row: its totals repeat the SASS rows below it
    try:
        e = float(x[iex] or 0)
        s = float(x[ist] or 0)
    except ValueError:
        continue
    name = "other"
    if cur_file != first_file:
        name = cur_file.rsplit("/", 1)[-1]
        if name not in [r[0] for r in ranges]:
            ranges.append((name, -1, -2))
    else:
        for n, lo, hi_ in ranges:
            if cur is not None and lo <= cur <= hi_:
                name = n
                break
    ins[name] += e
    stl[name] += s
ti = sum(ins.values()) or 1
ts = sum(stl.values()) or 1
print(f"total instructions {ti:.0f}")
for n in [r[0] for r in ranges] + ["other"]:
    print(f"{n:12s} {100 * ins[n] / ti:6.2f}% instr {100 * stl[n] / ts:6.2f}% stall  ({ins[n]:.0f})")
