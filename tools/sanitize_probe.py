#!/usr/bin/env python
"""Small workload that launches every kernel family of the library, for
compute-sanitizer (one tool per run; profiles/r02_sanitizer_*.txt):

    compute-sanitizer --tool memcheck  python tools/sanitize_probe.py
    compute-sanitizer --tool racecheck python tools/sanitize_probe.py
    compute-sanitizer --tool synccheck python tools/sanitize_probe.py

Covers: binning, rows + mirror, the fused cooperative rebuild (software grid
barrier), the pair pass, the row-based and the cell-based triplet passes
(window and shuffle forms: bases with |S+| below and above 32), C01
triplets and visit rows, the captured r-RESPA loop (drift, kick, fused
kick+drift, sample), the persistent ATM work counter, DirectSum, the RDF
histogram, and (--domain) a 2-rank decomposed run (ranks as processes
sharing cuda:0, gloo votes, ghosts pulled through CUDA IPC).
"""

from __future__ import annotations

import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "tests"))


def main(argv):
    import numpy as np
    import torch

    import paper_2507_11172_b200 as pkg
    from paper_2507_11172_b200 import observables
    from paper_2507_11172_b200.containers import collect_triplet_visits, engine_for
    from paper_2507_11172_b200.engine import ForceEngine

    done = []
    ff = pkg.ForceField(nu=0.073, cutoff=2.5)
    # container passes on both triplet forms (rc 3.0: |S+| > 32 bases too)
    for mode in ("0", "1"):
        ForceEngine.CELLS_MODE = mode
        for nc, rc3 in ((5, 2.5), (6, 3.0)):
            s = pkg.systems.fcc_system(nc, jitter=0.02, seed=5, temperature=0.9, vseed=6)
            f = pkg.ForceField(nu=0.073, cutoff=2.5, cutoff_3b=rc3)
            c = pkg.CudaLinkedCells()
            c.pair_pass(s, f)
            c.triplet_pass(s, f)
            done.append(f"passes cells={mode} nc={nc} rc3={rc3}: E3={c.triplet_energy:.6f}")
    ForceEngine.CELLS_MODE = "0"
    s = pkg.systems.fcc_system(5, jitter=0.02, seed=5)
    from types import SimpleNamespace

    rows = collect_triplet_visits(SimpleNamespace(cutoff=2.5), s)
    done.append(f"visit rows {len(rows)}")
    # device-resident r-RESPA: captured period graph, gated cooperative rebuild
    for mode in ("0", "1"):
        ForceEngine.CELLS_MODE = mode
        s = pkg.systems.fcc_system(6, jitter=0.02, seed=7, temperature=1.5, vseed=8)
        tr = pkg.respa_run(s, ff, pkg.CudaLinkedCells(), pkg.RespaSchedule(0.004, 5, 60))
        eng = engine_for(s.n)
        done.append(f"respa cells={mode}: rebuild steps {int(eng.status[3].item())}, "
                    f"E {tr.total[-1]:.6f}")
    ForceEngine.CELLS_MODE = "0"
    # DirectSum and RDF
    rng = np.random.default_rng(1)
    o = pkg.ParticleSystem.empty(64, np.array([8.0, 8.0, 8.0]), periodic=False)
    o.positions[:] = rng.uniform(0, 8, (64, 3))
    d = pkg.CudaDirectSum()
    d.pair_pass(o, ff)
    d.triplet_pass(o, ff)
    done.append(f"direct sum E3={d.triplet_energy:.6f}")
    s = pkg.systems.fcc_system(5, jitter=0.02, seed=5)
    h = observables.distance_histogram(torch.as_tensor(s.positions, device="cuda"), s.box,
                                       float(min(s.box)) / 2, 50)
    done.append(f"rdf counts {int(h.sum().item())}")
    if "--domain" in argv:
        import tempfile

        from test_gpu_parity import _run_domain_gpu

        with tempfile.TemporaryDirectory() as tmp:
            import pathlib

            out = _run_domain_gpu(pathlib.Path(tmp), 2, (2, 1, 1), "fcc", "peer")
            done.append(f"domain 2 ranks: x[0]={out['x'][0]}")
    torch.cuda.synchronize()
    print("\n".join(done))
    print("sanitize_probe ok")


if __name__ == "__main__":
    main(sys.argv[1:])
