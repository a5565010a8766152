#!/usr/bin/env python
"""Phase marks of the public respa_run on host arrays (bench.py's e2e leg).

    python tools/e2e_marks.py cfg2 20      # config, steps per call

Four calls of the same schedule: the first builds the cached run (rows
sized, period graph captured), the second captures the initial passes'
graph, the rest show the steady state.  Each line splits the call into its
marks (DeviceRespa.marks): before _drive ("pre"), start (upload + initial
passes enqueued), replays enqueued, the one synchronisation (collected),
the host copies (downloaded).
"""
import sys, time, os
sys.path.insert(0, os.getcwd())
import torch
import paper_2507_11172_b200 as pkg
from paper_2507_11172_b200 import integrators as I
from paper_2507_11172_b200.integrators import RespaSchedule
name = sys.argv[1]; steps = int(sys.argv[2])
cfg = pkg.systems.CONFIGS[name]
ff = cfg.force_field()
base = cfg.system()
for r in range(4):
    s = base.copy()
    torch.cuda.synchronize(); t0 = time.perf_counter()
    pkg.respa_run(s, ff, pkg.CudaLinkedCells(), RespaSchedule(cfg.dt, cfg.step_size_factor, steps))
    t1 = time.perf_counter()
    m = I.LAST_RUN[0].marks
    print(f"call {r}: {1e3*(t1-t0):.2f} ms", " | ".join(f"{m[i][0]} +{1e3*(m[i][1]-m[i-1][1]):.2f}" for i in range(1, len(m))), f"| end +{1e3*(t1-m[-1][1]):.2f}", f"| pre {1e3*(m[0][1]-t0):.2f}")
