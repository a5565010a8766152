#!/usr/bin/env python
"""DirectSum pass timings: all triplets / all pairs.

    python tools/direct_bench.py [N ...] [--reps R]

Random non-periodic systems at density ~0.5; CUDA-event medians of the
triplet pass (141 FP64 flops per triplet, the FP64 DFMA peak measured in the
same process) and the pair pass (35 flops per pair).  One JSON line per N.
"""

from __future__ import annotations

import ctypes
import json
import os
import statistics
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "tests"))


def main(argv):
    import numpy as np
    import torch

    from paper_2507_11172_b200 import _lib
    from paper_2507_11172_b200.engine import ForceEngine

    reps = 5
    if "--reps" in argv:
        reps = int(argv[argv.index("--reps") + 1])
        del argv[argv.index("--reps"): argv.index("--reps") + 2]
    sizes = [int(a) for a in argv] or [1024, 2048, 4096, 8192]
    L = _lib.lib()
    stream = _lib.stream_handle()
    peak = ctypes.c_double(0.0)
    L.rb_fp64_peak(2000, ctypes.byref(peak), stream)

    def timed(fn):
        fn()
        ts = []
        for _ in range(reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        return statistics.median(ts)

    for n in sizes:
        rng = np.random.default_rng(n)
        edge = (n / 0.5) ** (1.0 / 3.0)
        pos = rng.uniform(0.0, edge, (n, 3))  # overlaps are improbable at this density
        eng = ForceEngine(n)
        eng.upload_positions(pos)
        eng.reset_status(0)
        f = torch.empty((n, 3), dtype=torch.float64, device="cuda")
        t3 = timed(lambda: eng.direct_triplets(0.073, f))
        t2 = timed(lambda: eng.direct_pairs(1.0, 1.0, f, reduce=False))
        tri = n * (n - 1) * (n - 2) // 6
        pairs = n * (n - 1) // 2
        print(json.dumps({
            "n": n, "triplets": tri, "triplet_ms": t3, "triplets_per_s": tri / (t3 * 1e-3),
            "triplet_frac": tri * 141 / (t3 * 1e-3) / 1e12 / peak.value,
            "pairs": pairs, "pair_ms": t2, "pair_frac": pairs * 35 / (t2 * 1e-3) / 1e12 / peak.value,
            "fp64_peak_tflops": peak.value, "status": eng.read_status(),
        }), flush=True)


if __name__ == "__main__":
    main(sys.argv[1:])
