"""Host-side cell-grid geometry and stencil tables.

The device kernels need, per cutoff, the grid geometry and the canonical
neighbour-cell offsets; the functional API additionally exposes the triplet
offset patterns of the reference's ``CellGrid``.  Everything here is a pure
function of (box, extent, cutoff, periodic), evaluated in float64 exactly as
``respamd/containers.py`` does so that the device binning reproduces the
reference cell assignment bit for bit:

* geometry:        containers.py:244-262
* pair offsets:    containers.py:75-109, 133-144
* triplet patterns: containers.py:112-130, 147-172
"""

from __future__ import annotations

import functools
from dataclasses import dataclass
from typing import Optional

import numpy as np

from .model import ValidationError


@dataclass(frozen=True)
class Geometry:
    cells: tuple
    cell_size: tuple
    origin: tuple
    inv_cell: tuple
    reach: tuple
    cutoff: float
    periodic: bool
    box: tuple

    @property
    def num_cells(self) -> int:
        return int(np.prod(self.cells))


def geometry(box, positions: Optional[np.ndarray], cutoff: float, periodic: bool) -> Geometry:
    """Grid geometry (containers.py:244-262).

    Periodic grids need every box edge >= 2*cutoff (:248-252); open grids
    grow to cover drifted particles (:255-259), which needs the positions.
    """
    cutoff = float(cutoff)
    if cutoff <= 0:
        raise ValidationError(f"cutoff must be > 0, got {cutoff}")
    box = np.asarray(box, dtype=np.float64)
    if periodic:
        if np.any(box < 2.0 * cutoff):
            raise ValidationError(
                f"periodic box {box} too small for minimum-image safety at cutoff {cutoff}; "
                f"every edge must be >= {2.0 * cutoff}"
            )
        origin = np.zeros(3)
        extent = box.copy()
    else:
        lo = np.minimum(positions.min(axis=0), 0.0)
        hi = np.maximum(positions.max(axis=0) + 1e-9, box)
        origin = lo
        extent = hi - lo
    cells = np.maximum(1, np.floor(extent / cutoff).astype(np.int64))
    size = extent / cells
    reach = np.maximum(1, np.ceil(cutoff / size - 1e-12).astype(np.int64))
    inv = 1.0 / size
    return Geometry(
        cells=tuple(int(c) for c in cells), cell_size=tuple(float(s) for s in size),
        origin=tuple(float(o) for o in origin), inv_cell=tuple(float(v) for v in inv),
        reach=tuple(int(r) for r in reach), cutoff=cutoff, periodic=bool(periodic),
        box=tuple(float(b) for b in box),
    )


def _gap(delta, cells, size, periodic) -> float:
    """Minimal distance between two cells `delta` apart (containers.py:75-86)."""
    acc = 0.0
    for d in range(3):
        k = abs(int(delta[d]))
        if periodic:
            n = int(cells[d])
            k %= n
            k = min(k, n - k)
        g = max(0, k - 1) * float(size[d])
        acc += g * g
    return float(np.sqrt(acc))


def _cube(reach):
    rx, ry, rz = reach
    return [(x, y, z) for x in range(-rx, rx + 1) for y in range(-ry, ry + 1) for z in range(-rz, rz + 1)]


@functools.lru_cache(maxsize=64)
def _tables(cells, size, reach, cutoff, periodic):
    reachable = [o for o in _cube(reach) if _gap(o, cells, size, periodic) <= cutoff]
    raw = np.array(reachable, dtype=np.int64).reshape(-1, 3)
    pair = np.unique(np.mod(raw, np.asarray(cells)[None, :]), axis=0) if periodic else raw
    where = {tuple(int(v) for v in row): i for i, row in enumerate(pair)}

    def canon(o):
        return tuple(int(v) % int(n) for v, n in zip(o, cells)) if periodic else tuple(o)

    found = set()
    for c1 in reachable:
        for c2 in reachable:
            if c1 > c2:
                continue
            if _gap(tuple(b - a for a, b in zip(c1, c2)), cells, size, periodic) <= cutoff:
                i1, i2 = where[canon(c1)], where[canon(c2)]
                found.add((min(i1, i2), max(i1, i2)))
    patterns = np.array(sorted(found), dtype=np.int64).reshape(-1, 2)
    pair.flags.writeable = False
    patterns.flags.writeable = False
    return pair, patterns


def stencil(geom: Geometry):
    """(pair_cells (k,3) int64, triplet_patterns (p,2) int64, same_cell (p,) bool)."""
    pair, patterns = _tables(geom.cells, geom.cell_size, geom.reach, geom.cutoff, geom.periodic)
    return pair, patterns, patterns[:, 0] == patterns[:, 1]


def rb_grid(geom: Geometry):
    """The C-ABI ``rb_grid`` struct for this geometry."""
    from ._lib import RB_MAX_OFFSETS, RbGrid

    pair, _, _ = stencil(geom)
    if pair.shape[0] > RB_MAX_OFFSETS:
        raise ValidationError(f"{pair.shape[0]} neighbour offsets exceed {RB_MAX_OFFSETS}")
    g = RbGrid()
    for d in range(3):
        g.cells[d] = geom.cells[d]
        g.origin[d] = geom.origin[d]
        g.inv_cell[d] = geom.inv_cell[d]
        g.box[d] = geom.box[d]
    g.periodic = 1 if geom.periodic else 0
    g.n_offsets = int(pair.shape[0])
    for i, row in enumerate(pair):
        for d in range(3):
            g.offsets[i][d] = int(row[d])
    for d in range(3):
        g.wrap[d] = g.periodic
        g.gcells[d] = geom.cells[d]
        g.wlo[d] = 0
    return g


@dataclass(frozen=True)
class WindowGeometry:
    """A rank's window of a decomposed periodic grid (domain decomposition).

    ``base`` is the global periodic geometry; per dimension the local grid is
    either the whole wrapped dimension (``wrap[d]``, one rank along d) or the
    window of ``cells[d]`` global cells starting at global cell ``lo[d]``
    (the rank's block plus one halo layer on each side).  Distances keep the
    periodic minimum image of the whole box.
    """

    base: Geometry
    lo: tuple
    cells: tuple
    wrap: tuple

    @property
    def num_cells(self) -> int:
        return int(np.prod(self.cells))

    @property
    def cutoff(self) -> float:
        return self.base.cutoff

    @property
    def periodic(self) -> bool:
        return True

    @property
    def box(self) -> tuple:
        return self.base.box

    @property
    def cell_size(self) -> tuple:
        return self.base.cell_size

    def offsets(self) -> np.ndarray:
        """Neighbour offsets: canonical (mod n, deduplicated) in wrapped
        dimensions, raw -1/0/1 in windowed ones (the kernel skips cells
        outside the window)."""
        out = []
        for o in _cube((1, 1, 1)):
            t = tuple(int(v) % int(n) if w else int(v)
                      for v, n, w in zip(o, self.base.cells, self.wrap))
            if t not in out:
                out.append(t)
        return np.array(sorted(out), dtype=np.int64)

    def to_rb_grid(self):
        from ._lib import RbGrid

        offs = self.offsets()
        g = RbGrid()
        for d in range(3):
            g.cells[d] = self.cells[d]
            g.origin[d] = 0.0
            g.inv_cell[d] = self.base.inv_cell[d]
            g.box[d] = self.base.box[d]
            g.wrap[d] = 1 if self.wrap[d] else 0
            g.gcells[d] = self.base.cells[d]
            g.wlo[d] = self.lo[d]
        g.periodic = 1
        g.n_offsets = int(offs.shape[0])
        for i, row in enumerate(offs):
            for d in range(3):
                g.offsets[i][d] = int(row[d])
        return g


@dataclass
class CellGrid:
    """Host copy of one binning, field for field the reference ``CellGrid``
    (containers.py:50-72), produced by the device counting sort."""

    cells_per_dim: np.ndarray
    cell_size: np.ndarray
    origin: np.ndarray
    interaction_reach: np.ndarray
    cutoff: float
    periodic: bool
    box: np.ndarray
    cell_start: np.ndarray
    cell_particles: np.ndarray
    pair_cells: np.ndarray
    triplet_patterns: np.ndarray
    triplet_same_cell: np.ndarray

    @property
    def num_cells(self) -> int:
        return int(np.prod(self.cells_per_dim))

    def particles_of_cell(self, cell: int) -> np.ndarray:
        return self.cell_particles[self.cell_start[cell]: self.cell_start[cell + 1]]


