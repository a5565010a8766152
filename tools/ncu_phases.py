#!/usr/bin/env python
"""Instruction / stall shares of k_atm3 by phase (source-line ranges of
csrc/atm3.cu; lines inlined from common.cuh are reported as 'common').

    python tools/ncu_phases.py report.ncu-rep
"""
import collections
import csv
import os
import re
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(os.path.dirname(HERE), "paper_2507_11172_b200", "csrc", "atm3.cu")


def ranges():
    lines = open(SRC).read().splitlines()

    def find(pat, start=0):
        for i in range(start, len(lines)):
            if re.search(pat, lines[i]):
                return i + 1
        raise KeyError(pat)

    carve = find(r"A3Smem a3_carve\(")
    share = find(r"double owned_share\(")
    core = find(r"void a3_core\(")
    add = find(r"void a3_add\(")
    pair = find(r"void a3_eval\(")
    sub = find(r"void a3_add_j\(")
    win = find(r"void a3_windows\(")
    base = find(r"void a3_base\(")
    p0 = find(r"phase 0:")
    p1 = find(r"phase 1:")
    p3 = find(r"phase 3:")
    end = find(r"^}", p3)
    # (rsqrt_nr lives in common.cuh: reported under "common")
    return [("carve", carve, share - 1), ("owned share", share, core - 1),
            ("eval: ATM kernel", core, add - 1), ("slot accumulate", add, pair - 1),
            ("pair: accept + guard", pair, sub - 1), ("slot accumulate (sub-steps)", sub, win - 1),
            ("window loop", win, base - 1), ("setup", base, p0 - 1), ("phase 0 (S+ slots)", p0, p1 - 1),
            ("phase 1 call", p1, p3 - 1), ("phase 3 (write-back)", p3, end)]


def main(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv",
                          "--print-source=cuda,sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    cur_file, hdr, iex, ist = None, None, None, None
    tot_i = collections.Counter()
    tot_s = collections.Counter()
    rng = ranges()
    for x in rows:
        if x and x[0] == "File Path":
            cur_file = x[1]
            continue
        if x and x[0] == "Line No":
            hdr = x
            iex = hdr.index("Instructions Executed")
            ist = hdr.index("Warp Stall Sampling (All Samples)")
            continue
        # source-line rows only (their metrics aggregate the SASS rows below them)
        if hdr is None or not x or not x[0].isdigit() or len(x) <= max(iex, ist):
            continue
        ln = int(x[0])
        try:
            e = float(x[iex] or 0)
            s = float(x[ist] or 0)
        except ValueError:
            continue
        if cur_file and not cur_file.endswith("atm3.cu"):
            lab = "common (" + os.path.basename(cur_file) + ")"
        else:
            lab = next((n for n, lo, hi in rng if lo <= ln <= hi), "other")
        tot_i[lab] += e
        tot_s[lab] += s
    ti, ts = sum(tot_i.values()), sum(tot_s.values())
    print(f"total instructions {ti:.0f}")
    for lab, e in sorted(tot_i.items(), key=lambda kv: -kv[1]):
        print(f"  {lab:28s} {100 * e / ti:6.2f}% instr {100 * tot_s[lab] / ts:6.2f}% stall")


if __name__ == "__main__":
    main(sys.argv[1])
