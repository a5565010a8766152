#!/usr/bin/env python
"""Stall samples and instructions of an ncu report split by SASS region: the
innermost loops (backward branches) vs everything else, with the stall
reasons of each.

    python tools/ncu_regions.py report.ncu-rep
"""
import collections
import csv
import re
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hi = [i for i, x in enumerate(rows) if "Address" in x][0]
h = rows[hi]
data = [x for x in rows[hi + 1:] if len(x) == len(h)]
ia, isrc = h.index("Address"), h.index("Source")
iex = h.index("Instructions Executed")
reasons = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
ins = []
for x in data:
    try:
        a = int(x[ia], 16)
    except ValueError:
        continue
    ins.append((a, x[isrc], float(x[iex] or 0), {r: float(x[h.index(r)] or 0) for r in reasons}))
addr = {a: i for i, (a, *_rest) in enumerate(ins)}
loops = []
for i, (a, src, *_r) in enumerate(ins):
    m = re.search(r"BRA (0x[0-9a-f]+)", src)
    if m and "DIV" not in src:
        t = int(m.group(1), 16)
        if t < a and t in addr and 40 < i - addr[t] < 400:
            loops.append((addr[t], i))
inloop = set()
for lo, hi_ in loops:
    inloop.update(range(lo, hi_ + 1))
tot = collections.Counter()
agg = {"loops": collections.Counter(), "rest": collections.Counter()}
cnt = {"loops": 0.0, "rest": 0.0}
for i, (a, src, ex, st) in enumerate(ins):
    k = "loops" if i in inloop else "rest"
    cnt[k] += ex
    for r, v in st.items():
        agg[k][r] += v
        tot[r] += v
T = sum(tot.values())
for k in ("loops", "rest"):
    s = sum(agg[k].values())
    print(f"{k:6s} instr {cnt[k] / sum(cnt.values()):6.1%}  stall samples {s / T:6.1%}  top: " +
          ", ".join(f"{r[6:]} {v / T:.1%}" for r, v in agg[k].most_common(7)))
