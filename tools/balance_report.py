#!/usr/bin/env python
"""Estimated per-rank load of the domain decomposition (host only, no GPU).

    python tools/balance_report.py [cfg5] [--world 8]

Prints, for the even split of `auto_dims` and for the cost-aware layout of
`balanced_layout` (domain.py), the rank grid, the z boundaries, owned
particles per rank and the largest / mean estimated block cost (cell_costs:
pair work ~ neighbours, ATM work ~ neighbours^2 / s, plus the halo).
"""

from __future__ import annotations

import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def main(argv):
    import numpy as np

    from paper_2507_11172_b200 import systems
    from paper_2507_11172_b200.domain import (Decomposition, auto_dims, balanced_layout,
                                              block_costs, cell_costs, cell_occupancy)
    from paper_2507_11172_b200.grid import geometry

    world = int(argv[argv.index("--world") + 1]) if "--world" in argv else 8
    names = [a for a in argv if a.startswith("cfg")] or ["cfg5"]
    for name in names:
        cfg = systems.CONFIGS[name]
        system = cfg.system()
        ff = cfg.force_field()
        r_build = max(ff.cutoff, ff.cutoff_3b or ff.cutoff) + 0.3
        geom = geometry(system.box, None, r_build, True)
        costs = cell_costs(system.positions, geom, 0.29 / cfg.step_size_factor)
        occ = cell_occupancy(system.positions, geom)
        even_dims = auto_dims(world, geom.cells)
        even = Decomposition(system.box, r_build, world, 0, even_dims)
        dims, bounds = balanced_layout(costs, world, occ)
        for label, d, b in (("even", even_dims, even.bounds), ("balanced", dims, bounds)):
            load = block_costs(costs, d, b, occ)
            owners = Decomposition(system.box, r_build, world, 0, d, b).owner_rank(system.positions)
            counts = np.bincount(owners, minlength=world)
            print(f"{name} {label:8s} dims {d} z-bounds {list(map(int, b[2]))}  "
                  f"max/mean cost {load.max() / load.mean():.3f}  "
                  f"particles per rank {counts.min()}..{counts.max()}")


if __name__ == "__main__":
    main(sys.argv[1:])
