#!/usr/bin/env python
"""Per-kernel timings of the force passes on the BASELINE configs (step 0).

    python tools/kernel_bench.py [cfg2 cfg3 cfg4 ...] [--reps R] [--skin S]

For each config: bin + survivor rows once, then CUDA-event timings (median
of R, L2 flushed before each launch) of the LJ pass, the Newton-3 ATM pass
and the C01 ATM pass, with unique triplets/s and the FP64 fraction
(141 flops per unique triplet) against the DFMA peak
measured in the same process.  Prints one JSON object per config.
"""

from __future__ import annotations

import ctypes
import json
import os
import statistics
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def main(argv):
    import torch

    import paper_2507_11172_b200 as pkg
    from paper_2507_11172_b200 import _lib, grid
    from paper_2507_11172_b200.engine import ForceEngine

    reps = 10
    if "--reps" in argv:
        reps = int(argv[argv.index("--reps") + 1])
        del argv[argv.index("--reps"): argv.index("--reps") + 2]
    skin = 0.0
    if "--skin" in argv:  # Verlet rows at r_list + skin, as the device loop builds them
        skin = float(argv[argv.index("--skin") + 1])
        del argv[argv.index("--skin"): argv.index("--skin") + 2]
    names = argv or ["cfg2", "cfg3@2.0", "cfg3@2.5", "cfg3@3.0", "cfg4"]
    L = _lib.lib()
    stream = _lib.stream_handle()
    peak = ctypes.c_double(0.0)
    L.rb_fp64_peak(2000, ctypes.byref(peak), stream)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    def timed(fn):
        fn()
        ts = []
        for _ in range(reps):
            L.rb_l2_flush(_lib.ptr(flush), flush.numel(), stream)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        return statistics.median(ts)

    for name in names:
        cfg_name, _, rc3 = name.partition("@")
        cfg = pkg.systems.CONFIGS[cfg_name]
        rc3 = float(rc3) if rc3 else cfg.rc_atm
        s = cfg.system()
        r_list = max(cfg.rc_lj, rc3)
        eng = ForceEngine(s.n)
        r_build = r_list + skin
        geom = grid.geometry(s.box, None, r_build, True)
        eng.upload_positions(s.positions)
        eng.reset_status(0)
        eng.bin(geom)
        if skin > 0.0:  # slots as DeviceRespa.start sizes them
            eng.nlist(geom, rc3, checked=True)
            within = int(eng.max_count.item())
            eng.nlist(geom, r_build, capacity=None, checked=True)
            eng.slots = min(eng.capacity, (int(within * 1.25) + 8 + 31) // 32 * 32)
        else:
            eng.nlist(geom, r_list, checked=True)
        f = torch.empty((s.n, 3), dtype=torch.float64, device="cuda")
        eng.atm(geom, rc3, pkg.systems.NU, f, tag=0)
        torch.cuda.synchronize()
        unique = int(eng.visits.item())
        t_atm = timed(lambda: eng.atm_kernel(geom, rc3, pkg.systems.NU, f, 0))
        t_c01 = timed(lambda: eng.atm_c01(geom, rc3, pkg.systems.NU, f, 0, reduce=False))
        t_lj = timed(lambda: eng.lj_kernel(geom, cfg.rc_lj, 1.0, 1.0, f, 0))
        t_bin = timed(lambda: eng.bin(geom))
        t_nl = timed(lambda: eng.nlist(geom, r_build, capacity=eng.capacity, checked=False))
        # the fused gated rebuild of the device loop (bin + rows + mirror in
        # one launch), gate open (flag == tag 0) and closed
        eng.rebuild_flag.fill_(0)
        t_rb = timed(lambda: eng.rebuild(geom, r_build, eng.capacity, tag=0, fused=True))
        eng.rebuild_flag.fill_(-7)
        t_rb0 = timed(lambda: eng.rebuild(geom, r_build, eng.capacity, tag=0, fused=True))
        tps = unique / (t_atm * 1e-3)
        print(json.dumps({
            "config": name, "skin": skin, "n": s.n, "unique_triplets": unique, "capacity": eng.capacity,
            "slots": eng.slots, "atm_path": "cells" if eng.uses_cells(geom, rc3) else "rows",
            "nb_cap": eng.nb_cap, "cells_slots": eng.cells_slots(),
            "cells_smem": int(eng.L.rb_atm_cells_smem_bytes(int(eng.nb_cap or 32), eng.cells_slots())),
            "atm_ms": t_atm, "atm_c01_ms": t_c01, "lj_ms": t_lj,
            "bin_ms": t_bin, "nlist_ms": t_nl, "rebuild_ms": t_rb, "rebuild_closed_ms": t_rb0, "triplets_per_s": tps,
            "fp64_tflops": tps * 141 / 1e12, "fp64_peak_tflops": peak.value,
            "frac": tps * 141 / 1e12 / peak.value,
        }), flush=True)
        del eng


if __name__ == "__main__":
    main(sys.argv[1:])
