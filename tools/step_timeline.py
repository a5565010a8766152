#!/usr/bin/env python
"""Kernel timeline of the captured r-RESPA steps (bench.py's workload).

    python tools/step_timeline.py [cfg2] [--steps 50] [--flush]

Replays the per-step CUDA graphs under torch.profiler (CUPTI records every
kernel node of a graph) and prints, per kernel, launches / mean duration, and
per step the busy time (sum of kernel durations) against the span from the
first kernel start to the last kernel end -- the difference is the graph's
inter-node latency.  Not a bench number (profiler attached).
"""

from __future__ import annotations

import collections
import json
import os
import statistics
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def main(argv):
    import torch
    from torch.profiler import ProfilerActivity, profile

    import paper_2507_11172_b200 as pkg
    from paper_2507_11172_b200 import _lib
    from paper_2507_11172_b200.integrators import DeviceRespa, RespaSchedule

    steps = 50
    if "--steps" in argv:
        steps = int(argv[argv.index("--steps") + 1])
        del argv[argv.index("--steps"): argv.index("--steps") + 2]
    flush = "--flush" in argv
    argv = [a for a in argv if a != "--flush"]
    name = argv[0] if argv else "cfg2"
    cfg = pkg.systems.CONFIGS[name]
    sf = cfg.step_size_factor
    total = (sf + 10 + steps + 2 * sf + sf - 1) // sf * sf
    run = DeviceRespa(cfg.system(), cfg.force_field(), pkg.CudaLinkedCells(),
                      RespaSchedule(cfg.dt, sf, total), sf)
    run.start()
    run.run_periods(0, 1)
    graphs = run.capture_steps()
    step = sf
    for _ in range(10):
        graphs[step % sf].replay()
        step += 1
    L = _lib.lib()
    buf = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    torch.cuda.synchronize()
    marks = []
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(steps):
            if flush:
                L.rb_l2_flush(_lib.ptr(buf), buf.numel(), _lib.stream_handle())
            torch.cuda.synchronize()
            marks.append(step)
            graphs[step % sf].replay()
            torch.cuda.synchronize()
            step += 1
    path = "/tmp/rb_step_timeline.json"
    prof.export_chrome_trace(path)
    ev = [e for e in json.load(open(path))["traceEvents"]
          if e.get("cat") == "kernel" and e.get("ph") == "X"]
    ev.sort(key=lambda e: e["ts"])
    per = collections.defaultdict(list)
    for e in ev:
        per[e["name"].split("(")[0][:60]].append(e["dur"])
    print(f"{'kernel':60s} {'n':>5s} {'mean_us':>9s} {'total_us':>10s}")
    for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
        print(f"{k:60s} {len(v):5d} {statistics.mean(v):9.2f} {sum(v):10.1f}")
    # split into steps at the gaps introduced by the host synchronisation
    groups, cur = [], []
    for e in ev:
        if "k_flush" in e["name"]:
            continue
        if cur and e["ts"] - (cur[-1]["ts"] + cur[-1]["dur"]) > 50.0:
            groups.append(cur)
            cur = []
        cur.append(e)
    if cur:
        groups.append(cur)
    busy = [sum(e["dur"] for e in g) for g in groups]
    span = [g[-1]["ts"] + g[-1]["dur"] - g[0]["ts"] for g in groups]
    nk = [len(g) for g in groups]
    print(f"steps {len(groups)}: kernels/step {statistics.mean(nk):.1f}, busy {statistics.mean(busy):.1f} us, "
          f"span {statistics.mean(span):.1f} us, gaps {statistics.mean(span) - statistics.mean(busy):.1f} us")
    for j in range(sf):
        sel = [i for i, m in enumerate(marks[: len(groups)]) if m % sf == j]
        if sel:
            print(f"  position {j}: kernels {statistics.mean(nk[i] for i in sel):.1f} busy "
                  f"{statistics.mean(busy[i] for i in sel):.1f} span "
                  f"{statistics.mean(span[i] for i in sel):.1f}")


if __name__ == "__main__":
    main(sys.argv[1:])
