#!/usr/bin/env python
"""Per-step cost of the domain-decomposed loop on one GPU (world = 1).

    python tools/domain_probe.py [--config cfg4] [--steps K] [--backend nccl|gloo]

Runs domain_respa_run on a config (cfg2 default) with a single rank: no halo,
but every per-step piece of the multi-GPU loop (drift, rebuild vote,
refresh, passes, kicks, sample checks).  Prints ms/step (wall clock after a
warm-up run) next to the single-GPU graph loop's.
"""

from __future__ import annotations

import os
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def main(argv):
    import torch
    import torch.distributed as dist

    steps = int(argv[argv.index("--steps") + 1]) if "--steps" in argv else 200
    backend = argv[argv.index("--backend") + 1] if "--backend" in argv else "nccl"
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29533")
    torch.cuda.set_device(0)
    dist.init_process_group(backend, rank=0, world_size=1)
    import paper_2507_11172_b200 as pkg
    from paper_2507_11172_b200.domain_run import domain_respa_run, gpu_backend_factory

    cfg = pkg.systems.CONFIGS[argv[argv.index("--config") + 1] if "--config" in argv else "cfg2"]
    ff = cfg.force_field()
    sf = cfg.step_size_factor
    domain_respa_run(dist, cfg.system(), ff, pkg.RespaSchedule(cfg.dt, sf, 10),
                     gpu_backend_factory(ff))
    s = cfg.system()
    steps_run = {}

    def on_step(i):
        if i in (0, steps):
            torch.cuda.synchronize()
            steps_run[i] = time.perf_counter()

    prof = None
    if "--profile" in argv:
        import cProfile

        prof = cProfile.Profile()
        prof.enable()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    domain_respa_run(dist, s, ff, pkg.RespaSchedule(cfg.dt, sf, steps), gpu_backend_factory(ff),
                     on_step=on_step)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    if prof is not None:
        import pstats

        prof.disable()
        pstats.Stats(prof).sort_stats("tottime").print_stats(25)
        pstats.Stats(prof).sort_stats("cumtime").print_stats("paper_2507_11172_b200", 30)
    loop = steps_run[steps] - steps_run[0]
    from paper_2507_11172_b200.domain_run import WINDOW_STATS
    print(f"windows: {WINDOW_STATS}")
    print(f"domain loop (world 1, {backend}): {1e3 * dt / steps:.3f} ms/step over {steps} steps "
          f"incl. setup; step loop alone {1e3 * loop / steps:.3f} ms/step")
    s2 = cfg.system()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    pkg.respa_run(s2, ff, pkg.CudaLinkedCells(), pkg.RespaSchedule(cfg.dt, sf, steps))
    torch.cuda.synchronize()
    dt2 = time.perf_counter() - t0
    import numpy as np
    print(f"single-GPU respa_run: {1e3 * dt2 / steps:.3f} ms/step; max |dx| "
          f"{np.max(np.abs(s.positions - s2.positions)):.2e}")
    dist.destroy_process_group()


if __name__ == "__main__":
    main(sys.argv[1:])
