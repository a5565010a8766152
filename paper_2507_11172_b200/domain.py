"""Spatial domain decomposition of the periodic box over ranks.

One process per GPU.  The global periodic cell grid (cells >= r_build, the
row radius) is cut into a ``px x py x pz`` grid of blocks along cell
boundaries; a rank owns the particles whose global cell lies in its block
and keeps one halo layer of cells around it:

* migration (at row rebuilds): particles whose cell left the block go to the
  neighbouring rank, staged x -> y -> z so diagonal moves need no extra
  messages;
* ghosts (at row rebuilds): the first/last cell layer of the block is sent
  to the -/+ neighbour, staged x -> y -> z with the ghosts of earlier stages
  included, which fills edges and corners; the send lists are kept;
* every step: the same lists carry the owners' new positions to the ghosts.

Forces are owner-computes across ranks: every triplet/pair containing an
owned particle has all its members in owned + ghosts (they are within the
cutoff of that particle), so the local passes give complete forces on owned
particles and no reverse communication is needed; ghost forces are dropped.
Energies are attributed phi/2 per owned pair member and phi/3 per owned
triplet member (the reference's C01 attribution, containers.py:364, :524),
so per-rank partials sum to the global scalars; they are summed in rank
order (deterministic).

The exchange runs on torch.distributed point-to-point (NCCL between GPUs,
gloo for the CPU tests) and is independent of the force backend, which is
the sm_100a engine in production and a numpy reference in the tests.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from .grid import Geometry, WindowGeometry, geometry

PAYLOAD = 13  # id, x(3), v(3), f2_old(3), f3(3)


def auto_dims(world: int, cells) -> tuple:
    """Rank grid: the factorisation of `world` with the most cubic blocks
    among those leaving every split block at least one cell plus a halo."""
    best, best_score = None, None
    for px in range(1, world + 1):
        if world % px:
            continue
        for py in range(1, world // px + 1):
            if (world // px) % py:
                continue
            dims = (px, py, world // px // py)
            ok = all(p == 1 or (c // p >= 1 and -(-c // p) + 2 <= c) for c, p in zip(cells, dims))
            if not ok:
                continue
            blk = [c / p for c, p in zip(cells, dims)]
            score = max(blk) / min(blk)
            if best is None or score < best_score - 1e-12:
                best, best_score = dims, score
    if best is None:
        raise ValueError(f"cannot decompose {cells} cells over {world} ranks")
    return best


# ---------------------------------------------------------------------------
# cost-aware block boundaries (inhomogeneous systems, e.g. the cfg5 slab)
# ---------------------------------------------------------------------------


def cell_occupancy(positions: np.ndarray, geom: Geometry) -> np.ndarray:
    """Particles per global cell (the binning arithmetic), shape `geom.cells`."""
    n = np.asarray(geom.cells)
    inv = np.asarray(geom.inv_cell)
    c = np.clip(np.trunc(np.asarray(positions) * inv[None, :]).astype(np.int64), 0, n[None, :] - 1)
    occ = np.zeros(tuple(n), dtype=np.float64)
    np.add.at(occ, (c[:, 0], c[:, 1], c[:, 2]), 1.0)
    return occ


def cell_costs(positions: np.ndarray, geom: Geometry, triplet_weight: float = 0.0) -> np.ndarray:
    """Estimated work per global cell, shape `geom.cells`.

    A particle's pair work grows with its neighbour count, its triplet work
    with the square of it; the neighbour count is estimated from the
    occupancy of the 27 surrounding cells (cells >= r_build, so the cutoff
    sphere fills ~0.155 of them).  Per particle: 5 (integration, binning,
    rows) + nb + triplet_weight * nb^2, with triplet_weight ~ 0.29 / s for
    the ATM pass every s-th step (4x the flops of a pair, 210 triplets per
    54 pairs in the rho 0.8 liquid).  A heuristic: it only moves block
    boundaries, never results."""
    occ = cell_occupancy(positions, geom)
    around = np.zeros_like(occ)
    for a in (-1, 0, 1):
        for b in (-1, 0, 1):
            for e in (-1, 0, 1):
                around += np.roll(occ, (a, b, e), axis=(0, 1, 2))
    nb = 0.155 * around
    return occ * (5.0 + nb + float(triplet_weight) * nb * nb)


def balanced_bounds(profile: np.ndarray, parts: int) -> np.ndarray:
    """Cut a periodic row of cell layers into `parts` contiguous blocks
    (boundaries at 0 and n) minimising the largest block cost; every block
    keeps >= 1 layer and, when split, leaves room for its two halo layers
    (width <= n - 2).  Exact DP, ties to the leftmost cut (deterministic)."""
    profile = np.asarray(profile, dtype=np.float64)
    n = profile.shape[0]
    if parts == 1:
        return np.array([0, n])
    cum = np.concatenate([[0.0], np.cumsum(profile)])
    w_max = n - 2
    inf = float("inf")
    # best[p][e]: minimal max cost of splitting layers [0, e) into p blocks
    best = np.full((parts + 1, n + 1), inf)
    cut = np.zeros((parts + 1, n + 1), dtype=np.int64)
    best[0][0] = 0.0
    for p in range(1, parts + 1):
        for e in range(p, n + 1):
            for b in range(max(p - 1, e - w_max), e):
                if best[p - 1][b] == inf:
                    continue
                v = max(best[p - 1][b], cum[e] - cum[b])
                if v < best[p][e]:
                    best[p][e], cut[p][e] = v, b
    if best[parts][n] == inf:
        raise ValueError(f"cannot cut {n} cell layers into {parts} blocks with halos")
    bounds = [n]
    for p in range(parts, 0, -1):
        bounds.append(int(cut[p][bounds[-1]]))
    return np.array(bounds[::-1])


def block_costs(costs: np.ndarray, dims, bounds, occ: Optional[np.ndarray] = None,
                ghost_cost: float = 5.0) -> np.ndarray:
    """Cost per block of the rank grid (rank order): the block's cells, plus
    `ghost_cost` per particle of its halo layer (split dimensions, periodic)
    when the occupancy `occ` is given."""
    n = costs.shape
    out = []
    for bx in range(dims[0]):
        for by in range(dims[1]):
            for bz in range(dims[2]):
                ks = (bx, by, bz)
                own = np.ix_(*[np.arange(bounds[d][ks[d]], bounds[d][ks[d] + 1])
                               for d in range(3)])
                total = float(costs[own].sum())
                if occ is not None:
                    win = np.ix_(*[np.arange(bounds[d][ks[d]] - 1, bounds[d][ks[d] + 1] + 1) % n[d]
                                   if dims[d] > 1 else np.arange(n[d]) for d in range(3)])
                    total += ghost_cost * float(occ[win].sum() - occ[own].sum())
                out.append(total)
    return np.array(out)


def balanced_layout(costs: np.ndarray, world: int, occ: Optional[np.ndarray] = None):
    """(dims, bounds) for a cost array: every factorisation of `world` whose
    blocks can hold a halo, each dimension cut by `balanced_bounds` on its
    cost profile; the layout with the smallest largest-block cost (ghosts
    included when `occ` is given) wins, ties within 1e-9 relative to the
    most cubic blocks, as `auto_dims`."""
    n = costs.shape
    best = None
    for px in range(1, world + 1):
        if world % px:
            continue
        for py in range(1, world // px + 1):
            if (world // px) % py:
                continue
            dims = (px, py, world // px // py)
            try:
                bounds = [balanced_bounds(costs.sum(axis=tuple(a for a in range(3) if a != d)),
                                          dims[d]) for d in range(3)]
            except ValueError:
                continue
            worst = float(block_costs(costs, dims, bounds, occ).max())
            blk = [c / p for c, p in zip(n, dims)]
            shape = max(blk) / min(blk)
            key = (worst, shape)
            if best is None or key[0] < best[0][0] * (1 - 1e-9) or \
                    (key[0] <= best[0][0] * (1 + 1e-9) and shape < best[0][1] - 1e-12):
                best = (key, dims, bounds)
    if best is None:
        raise ValueError(f"cannot decompose {n} cells over {world} ranks")
    return best[1], best[2]


@dataclass
class Decomposition:
    """Block geometry of one rank.  `bounds` (optional, per dimension the
    dims[d] + 1 cell boundaries from 0 to cells[d]) replaces the even split,
    e.g. with `balanced_layout`'s cost-aware cuts."""

    box: np.ndarray
    r_build: float
    world: int
    rank: int
    dims: Optional[tuple] = None
    bounds: Optional[list] = None
    geom: Geometry = field(init=False)

    def __post_init__(self):
        self.box = np.asarray(self.box, dtype=np.float64)
        self.geom = geometry(self.box, None, self.r_build, True)
        n = self.geom.cells
        if self.dims is None:
            self.dims = auto_dims(self.world, n)
        self.dims = tuple(int(p) for p in self.dims)
        if int(np.prod(self.dims)) != self.world:
            raise ValueError(f"rank grid {self.dims} does not match world size {self.world}")
        px, py, pz = self.dims
        self.coord = (self.rank // (py * pz), (self.rank // pz) % py, self.rank % pz)
        if self.bounds is None:
            self.bounds = [np.array([k * n[d] // self.dims[d] for k in range(self.dims[d] + 1)])
                           for d in range(3)]
        else:
            self.bounds = [np.asarray(b, dtype=np.int64) for b in self.bounds]
            for d in range(3):
                b = self.bounds[d]
                if b.shape != (self.dims[d] + 1,) or b[0] != 0 or b[-1] != n[d] or \
                        np.any(np.diff(b) < 1):
                    raise ValueError(f"bad block bounds {b.tolist()} for {n[d]} cells / "
                                     f"{self.dims[d]} blocks in dim {d}")
        self.lo = tuple(int(self.bounds[d][self.coord[d]]) for d in range(3))
        self.hi = tuple(int(self.bounds[d][self.coord[d] + 1]) for d in range(3))
        for d in range(3):
            if self.dims[d] > 1 and (self.hi[d] - self.lo[d] < 1 or
                                     self.hi[d] - self.lo[d] + 2 > n[d]):
                raise ValueError(f"block {self.lo}-{self.hi} too thin for a halo in dim {d}")

    # ----------------------------------------------------------- topology
    def split(self, d: int) -> bool:
        return self.dims[d] > 1

    def neighbor(self, d: int, step: int) -> int:
        c = list(self.coord)
        c[d] = (c[d] + step) % self.dims[d]
        return (c[0] * self.dims[1] + c[1]) * self.dims[2] + c[2]

    def window(self) -> WindowGeometry:
        n = self.geom.cells
        lo, cells, wrap = [], [], []
        for d in range(3):
            if self.split(d):
                lo.append((self.lo[d] - 1) % n[d])
                cells.append(self.hi[d] - self.lo[d] + 2)
                wrap.append(False)
            else:
                lo.append(0)
                cells.append(n[d])
                wrap.append(True)
        return WindowGeometry(self.geom, tuple(lo), tuple(cells), tuple(wrap))

    # ------------------------------------------------------- cell indices
    def cells_of(self, pos: np.ndarray) -> np.ndarray:
        """Global cell index per particle and dimension: the binning
        arithmetic of containers.py:182-196 (truncation, clamp)."""
        inv = np.asarray(self.geom.inv_cell)
        n = np.asarray(self.geom.cells)
        c = np.trunc(pos * inv[None, :]).astype(np.int64)
        return np.clip(c, 0, n[None, :] - 1)

    def cells_of_t(self, pos):
        """cells_of on a torch tensor (on its device; the same IEEE
        arithmetic: one product, truncation, clamp)."""
        import torch

        inv = torch.tensor(self.geom.inv_cell, dtype=torch.float64, device=pos.device)
        n = torch.tensor(self.geom.cells, dtype=torch.int64, device=pos.device)
        c = torch.trunc(pos * inv[None, :]).to(torch.int64)
        return torch.minimum(torch.clamp(c, min=0), n[None, :] - 1)

    def block_coord_t(self, cells_d, d: int):
        """Block coordinate along dimension d of global cell indices (torch)."""
        import torch

        b = torch.as_tensor(np.asarray(self.bounds[d], dtype=np.int64), device=cells_d.device)
        return torch.searchsorted(b, cells_d.contiguous(), right=True) - 1

    def block_of(self, cells: np.ndarray) -> np.ndarray:
        """Block coordinate per particle and dimension."""
        out = np.empty_like(cells)
        for d in range(3):
            out[:, d] = np.searchsorted(self.bounds[d], cells[:, d], side="right") - 1
        return out

    def window_count(self, pos: np.ndarray) -> int:
        """Particles whose cell lies in this rank's block or halo layer
        (owned + ghosts right after a rebuild)."""
        c = self.cells_of(np.asarray(pos))
        inside = np.ones(c.shape[0], dtype=bool)
        n = self.geom.cells
        for d in range(3):
            if self.split(d):
                rel = (c[:, d] - self.lo[d] + 1) % n[d]
                inside &= rel < self.hi[d] - self.lo[d] + 2
        return int(inside.sum())

    def window_count_t(self, pos) -> int:
        """window_count on a torch tensor (on its device)."""
        import torch

        c = self.cells_of_t(pos)
        inside = torch.ones(c.shape[0], dtype=torch.bool, device=pos.device)
        n = self.geom.cells
        for d in range(3):
            if self.split(d):
                rel = torch.remainder(c[:, d] - self.lo[d] + 1, n[d])
                inside &= rel < self.hi[d] - self.lo[d] + 2
        return int(inside.sum().item())

    def owner_rank_t(self, pos):
        """owner_rank on a torch tensor (on its device)."""
        c = self.cells_of_t(pos)
        b = [self.block_coord_t(c[:, d], d) for d in range(3)]
        return (b[0] * self.dims[1] + b[1]) * self.dims[2] + b[2]

    def owner_rank(self, pos: np.ndarray) -> np.ndarray:
        b = self.block_of(self.cells_of(pos))
        return (b[:, 0] * self.dims[1] + b[:, 1]) * self.dims[2] + b[:, 2]


# ---------------------------------------------------------------------------
# point-to-point exchange (torch.distributed; gloo or NCCL)
# ---------------------------------------------------------------------------


class Exchanger:
    """Two-phase neighbour exchange along one dimension: phase 1 sends to the
    - neighbour and receives from the + neighbour, phase 2 the reverse.  Works
    for a two-rank ring (both neighbours the same rank)."""

    def __init__(self, dist, device):
        import torch

        self.dist = dist
        self.device = torch.device(device)
        # gloo moves host tensors only: stage device tensors through the host
        self.wire = (torch.device("cpu") if dist.get_backend() == "gloo" else self.device)

    def _pair(self, send, dst, src, width, dtype):
        import torch

        dist = self.dist
        send = send.to(self.wire)
        n_send = torch.tensor([send.shape[0]], dtype=torch.int64, device=self.wire)
        n_recv = torch.zeros(1, dtype=torch.int64, device=self.wire)
        reqs = dist.batch_isend_irecv([dist.P2POp(dist.isend, n_send, dst),
                                       dist.P2POp(dist.irecv, n_recv, src)])
        for r in reqs:
            r.wait()
        recv = torch.empty((int(n_recv.item()), width), dtype=dtype, device=self.wire)
        ops = []
        if send.shape[0]:
            ops.append(dist.P2POp(dist.isend, send.contiguous(), dst))
        if recv.shape[0]:
            ops.append(dist.P2POp(dist.irecv, recv, src))
        if ops:
            for r in dist.batch_isend_irecv(ops):
                r.wait()
        return recv.to(self.device)

    def exchange(self, to_minus, to_plus, minus: int, plus: int):
        """Returns (from_plus, from_minus)."""
        width, dtype = to_minus.shape[1], to_minus.dtype
        from_plus = self._pair(to_minus, minus, plus, width, dtype)
        from_minus = self._pair(to_plus, plus, minus, width, dtype)
        return from_plus, from_minus

    def exchange_fixed(self, to_minus, to_plus, minus: int, plus: int, n_from_plus: int,
                       n_from_minus: int):
        """Same with known receive sizes (per-step ghost refresh: one round)."""
        import torch

        dist = self.dist
        width, dtype = to_minus.shape[1], to_minus.dtype
        from_plus = torch.empty((n_from_plus, width), dtype=dtype, device=self.wire)
        from_minus = torch.empty((n_from_minus, width), dtype=dtype, device=self.wire)
        for send, dst, recv, src in ((to_minus.to(self.wire), minus, from_plus, plus),
                                     (to_plus.to(self.wire), plus, from_minus, minus)):
            ops = []
            if send.shape[0]:
                ops.append(dist.P2POp(dist.isend, send.contiguous(), dst))
            if recv.shape[0]:
                ops.append(dist.P2POp(dist.irecv, recv, src))
            if ops:
                for r in dist.batch_isend_irecv(ops):
                    r.wait()
        return from_plus.to(self.device), from_minus.to(self.device)


# ---------------------------------------------------------------------------
# migration and ghosts
# ---------------------------------------------------------------------------


@dataclass
class GhostPlan:
    """Send lists of the staged ghost exchange, replayed every step."""

    stages: list  # per split dimension: (d, idx_to_minus, idx_to_plus, n_from_plus, n_from_minus)
    n_owned: int
    n_local: int
    origin: object = None  # (n_local, 2) owner rank, owner row (build_ghosts(origin=...))


def migrate(dec: Decomposition, ex: Exchanger, payload):
    """Move owned particles whose cell left the block to their new owner.

    `payload` is an (n, PAYLOAD) float64 tensor: id, x, v, f2_old, f3.
    Staged x -> y -> z; a particle moves at most one block per rebuild
    (the skin bounds the displacement)."""
    import torch

    if not any(dec.split(d) for d in range(3)):
        return payload  # one block: nothing moves, the order (ascending id) stands
    for d in range(3):
        if not dec.split(d):
            continue
        # cell and block maps on the payload's device (no host round trip of
        # the positions)
        blk = dec.block_coord_t(dec.cells_of_t(payload[:, 1:4])[:, d], d)
        me, p = dec.coord[d], dec.dims[d]
        stay = blk == me
        to_minus = (~stay) & (blk == (me - 1) % p)
        to_plus = (~stay) & (~to_minus)
        if bool(torch.any(to_plus & (blk != (me + 1) % p))):
            raise RuntimeError("a particle moved more than one block between row rebuilds")
        from_plus, from_minus = ex.exchange(payload[to_minus], payload[to_plus],
                                            dec.neighbor(d, -1), dec.neighbor(d, +1))
        payload = torch.cat([payload[stay], from_plus, from_minus], dim=0)
    # deterministic local order: ascending global id
    order = torch.argsort(payload[:, 0])
    return payload[order]


def build_ghosts(dec: Decomposition, ex: Exchanger, pos_owned, origin=None):
    """Staged ghost exchange; returns (local positions (owned first), plan).

    With `origin` ((n_own, 2) float64: owner rank, owner row per owned row)
    the messages carry it along and the plan's `origin` holds it for every
    local row: where a ghost's position lives at its owner (the pull lists
    of the peer-memory refresh)."""
    import torch

    n_own = int(pos_owned.shape[0])
    local = pos_owned if origin is None else torch.cat([pos_owned, origin], dim=1)
    stages = []
    for d in range(3):
        if not dec.split(d):
            continue
        cells = dec.cells_of_t(local[:, :3])[:, d]
        tm = torch.nonzero(cells == dec.lo[d]).reshape(-1)
        tp = torch.nonzero(cells == dec.hi[d] - 1).reshape(-1)
        from_plus, from_minus = ex.exchange(local[tm], local[tp], dec.neighbor(d, -1),
                                            dec.neighbor(d, +1))
        stages.append((d, tm, tp, int(from_plus.shape[0]), int(from_minus.shape[0])))
        local = torch.cat([local, from_plus, from_minus], dim=0)
    plan = GhostPlan(stages, n_own, int(local.shape[0]))
    if origin is not None:
        plan.origin = local[:, 3:5]
        local = local[:, 0:3].contiguous()
    return local, plan


def refresh_ghosts(dec: Decomposition, ex: Exchanger, plan: GhostPlan, local):
    """Per step: the owners' new positions into the ghost slots (in place)."""
    at = plan.n_owned
    for d, tm, tp, n_fp, n_fm in plan.stages:
        from_plus, from_minus = ex.exchange_fixed(local[tm], local[tp], dec.neighbor(d, -1),
                                                  dec.neighbor(d, +1), n_fp, n_fm)
        local[at:at + n_fp] = from_plus
        local[at + n_fp:at + n_fp + n_fm] = from_minus
        at += n_fp + n_fm
    return local


def allsum_in_rank_order(dist, values, device):
    """Sum a small vector over ranks in rank order (deterministic)."""
    import torch

    wire = torch.device("cpu") if dist.get_backend() == "gloo" else torch.device(device)
    t = torch.as_tensor(np.asarray(values, dtype=np.float64), device=wire)
    parts = [torch.empty_like(t) for _ in range(dist.get_world_size())]
    dist.all_gather(parts, t)
    acc = np.zeros_like(np.asarray(values, dtype=np.float64))
    for p in parts:
        acc = acc + p.cpu().numpy()
    return acc
