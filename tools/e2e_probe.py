#!/usr/bin/env python
"""Where the wall time of the public respa_run goes (bench.py's e2e leg).

    python tools/e2e_probe.py [cfg2] [--steps 1000] [--reps 5]

Times respa_run end to end `reps` times, then one run split into its phases
(DeviceRespa construction, start, eager first period, capture, replays,
download) with a device synchronisation around each.
"""

from __future__ import annotations

import os
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def main(argv):
    import torch

    import paper_2507_11172_b200 as pkg
    from paper_2507_11172_b200.integrators import DeviceRespa, RespaSchedule

    def opt(name, default):
        if name in argv:
            v = int(argv[argv.index(name) + 1])
            del argv[argv.index(name): argv.index(name) + 2]
            return v
        return default

    steps, reps = opt("--steps", 1000), opt("--reps", 5)
    cfg = pkg.systems.CONFIGS[argv[0] if argv else "cfg2"]
    sf = cfg.step_size_factor
    ff = cfg.force_field()
    for r in range(reps):
        s = cfg.system()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        pkg.respa_run(s, ff, pkg.CudaLinkedCells(), RespaSchedule(cfg.dt, sf, steps))
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        print(f"respa_run {steps} steps: {dt * 1e3:8.1f} ms  ({steps / dt:8.0f} steps/s)")

    def tick(label, t):
        torch.cuda.synchronize()
        now = time.perf_counter()
        print(f"  {label:24s} {1e3 * (now - t):8.2f} ms")
        return now

    s = cfg.system()
    t = time.perf_counter()
    run = DeviceRespa(s, ff, pkg.CudaLinkedCells(), RespaSchedule(cfg.dt, sf, steps), sf)
    t = tick("construct", t)
    run.start()
    t = tick("start", t)
    run.run_periods(0, 1)
    t = tick("first period (eager)", t)
    run.capture()
    t = tick("capture", t)
    run.eng.set_step(run.interval)
    t = tick("status reset", t)
    n_periods = steps // run.interval
    run.run_periods(1, n_periods - 1)
    t = tick(f"replay {n_periods - 1} periods", t)
    run.finish_scalars()
    rows = run.trace_rows(n_periods + 1)
    t = tick("finish + trace", t)
    run.download()
    t = tick("download", t)
    print(f"  rows {rows.shape}, status {run.eng.read_status()}")


if __name__ == "__main__":
    main(sys.argv[1:])
