"""DirectSum distributed over ranks.

The paper distributes its all-pairs/all-triplets reference over MPI ranks
with a communication-reducing three-body scheme.  Here the particle data of
a DirectSum (n <= 8192: 200 KB of positions) is replicated on every rank and
the WORK is split: rank r evaluates the pairs of its particle range and the
triplets whose lowest member lies in its base range -- base ranges cut so
that every rank gets the same number of triplets (base i owns
(n-1-i)(n-2-i)/2 of them).  One all-gather of the partial forces and scalars
per pass, summed in rank order: every rank ends with the same, deterministic
result.  The kernels are rb_direct_pairs_range / rb_direct_triplets_range.
"""

from __future__ import annotations

import numpy as np

from .containers import _DIRECT_PERIODIC_MSG, _raise_on_status, engine_for
from .engine import SCALAR_E2, SCALAR_E3, SCALAR_W2, SCALAR_W3
from .model import ValidationError


def particle_ranges(n: int, parts: int) -> list:
    """Equal particle ranges (the pair pass: every particle costs n - 1 pairs)."""
    return [(n * r // parts, n * (r + 1) // parts) for r in range(parts)]


def base_ranges(n: int, parts: int) -> list:
    """Base-particle ranges with equal triplet counts (base i owns
    C(n-1-i, 2) triplets): cuts at the 1/parts quantiles of the cumulative
    count."""
    m = np.arange(n - 1, -1, -1, dtype=np.float64)  # followers of base i
    work = np.cumsum(m * (m - 1) / 2.0)
    total = work[-1] if n else 0.0
    cuts = [0]
    for r in range(1, parts):
        cuts.append(int(np.searchsorted(work, total * r / parts, side="left")) + 1 if total else 0)
    cuts.append(n)
    cuts = [min(max(c, 0), n) for c in cuts]
    for r in range(1, len(cuts)):
        cuts[r] = max(cuts[r], cuts[r - 1])
    return [(cuts[r], cuts[r + 1]) for r in range(parts)]


class DistributedDirectSum:
    """DirectSum container over the ranks of `dist` (torch.distributed):
    the duck type of ``respamd.containers.DirectSum``; call the passes on
    every rank with the same system."""

    name = "cuda_direct_sum_distributed"

    def __init__(self, dist):
        self.dist = dist
        self.pair_energy = self.pair_virial = 0.0
        self.triplet_energy = self.triplet_virial = 0.0

    def _combine(self, forces, e, w):
        """All-gather (forces, e, w) of every rank; sum in rank order."""
        import torch

        dist = self.dist
        wire = torch.device("cpu") if dist.get_backend() == "gloo" else forces.device
        mine = torch.cat([forces.reshape(-1), torch.stack([e, w])]).to(wire)
        parts = [torch.empty_like(mine) for _ in range(dist.get_world_size())]
        dist.all_gather(parts, mine)
        acc = parts[0].clone()
        for p in parts[1:]:
            acc += p
        out = acc.cpu().numpy()
        n3 = forces.numel()
        return out[:n3].reshape(-1, 3), float(out[n3]), float(out[n3 + 1])

    def _engine(self, system):
        if system.periodic:
            raise ValidationError(_DIRECT_PERIODIC_MSG)
        eng = engine_for(system.positions.shape[0])
        eng.upload_positions(system.positions)
        eng.reset_status(0)
        return eng

    def pair_pass(self, system, ff) -> None:
        eng = self._engine(system)
        torch, n = eng.torch, eng.n
        lo, hi = particle_ranges(n, self.dist.get_world_size())[self.dist.get_rank()]
        out = torch.zeros((n, 3), dtype=torch.float64, device=eng.device)
        eng.e2_rank.zero_()
        eng.w2_rank.zero_()
        eng.direct_pairs(ff.epsilon, ff.sigma, out, tag=0, rng=(lo, hi))
        _raise_on_status(eng)
        f, self.pair_energy, self.pair_virial = self._combine(
            out, eng.scalars[SCALAR_E2], eng.scalars[SCALAR_W2])
        system.forces_2b[:] = f

    def triplet_pass(self, system, ff) -> None:
        if ff.nu == 0.0:
            system.forces_3b[:] = 0.0
            self.triplet_energy = self.triplet_virial = 0.0
            return
        eng = self._engine(system)
        torch, n = eng.torch, eng.n
        lo, hi = base_ranges(n, self.dist.get_world_size())[self.dist.get_rank()]
        out = torch.empty((n, 3), dtype=torch.float64, device=eng.device)
        eng.direct_triplets(ff.nu, out, tag=0, rng=(lo, hi))
        _raise_on_status(eng)
        f, self.triplet_energy, self.triplet_virial = self._combine(
            out, eng.scalars[SCALAR_E3], eng.scalars[SCALAR_W3])
        system.forces_3b[:] = f


__all__ = ["DistributedDirectSum", "base_ranges", "particle_ranges"]
