"""Drop-in GPU container and functional passes (the reference's L2 boundary).

``CudaLinkedCells`` has the exact duck type of ``respamd.containers.LinkedCells``
(containers.py:878-937): a ``name``, the four scalars of the most recent
passes, and ``pair_pass(system, ff)`` / ``triplet_pass(system, ff)`` that
overwrite ``system.forces_2b`` / ``system.forces_3b`` in place and raise
``MinimumSeparationError`` when two particles come closer than the guard.
It works with the reference's own ``ParticleSystem``/``ForceField`` objects
and with this package's mirrors, and plugs into the reference's
``respa_run`` unchanged (host arrays are copied to HBM and back per pass) or
into this package's device-resident :func:`integrators.respa_run`.

The functional mirrors (``build_cell_grid``, ``c01_pair_pass``,
``c01_triplet_pass``, ``collect_triplet_visits``) return reference-layout
results (int64 cell tables, ``(forces, energy, virial)`` tuples) so the
reference's own tests can be pointed at the GPU path.

All arithmetic runs in the sm_100a kernels; there is no CPU fallback.
"""

from __future__ import annotations

from typing import Optional

import numpy as np

from . import grid as _grid
from .engine import ForceEngine, SCALAR_E2, SCALAR_E3, SCALAR_W2, SCALAR_W3
from .model import ValidationError, triplet_cutoff


class MinimumSeparationError(ValidationError):
    """Two particles came closer than the kernel separation guard
    (``respamd/containers.py:39-40``)."""


_MINSEP_MSG = ("particles closer than the minimum separation guard; the configuration is "
               "(nearly) singular")

_ENGINES: dict = {}


def engine_for(n: int, run: bool = False) -> ForceEngine:
    """Per-particle-count device workspace, reused across passes.

    A device-resident run keeps its state (rows, x_ref, status) in its
    engine between steps; while one holds the workspace (``busy``), container
    passes -- e.g. a host hook calling ``pair_pass`` -- get a second one, so
    they never disturb the run's skin invariant or its pending errors.
    ``run=True``: the caller is such a run (and takes the primary engine)."""
    key = (n, False)
    eng = _ENGINES.get(key)
    if eng is not None and eng.busy and not run:
        key = (n, True)
        eng = _ENGINES.get(key)
    if eng is None:
        if len(_ENGINES) > 8:
            _ENGINES.clear()
        eng = ForceEngine(n)
        _ENGINES[key] = eng
    return eng


def _geometry_for(system, cutoff) -> _grid.Geometry:
    pos = None if system.periodic else np.asarray(system.positions, dtype=np.float64)
    return _grid.geometry(system.box, pos, cutoff, bool(system.periodic))


def _prepare(system, cutoff):
    """Upload positions, bin and build survivor rows within `cutoff`."""
    eng = engine_for(system.positions.shape[0])
    geom = _geometry_for(system, cutoff)
    eng.upload_positions(system.positions)
    eng.reset_status(0)
    eng.bin(geom)
    eng.nlist(geom, geom.cutoff, capacity=None, checked=True)
    eng.nb_cap = 0  # the cell-based triplet pass re-measures its neighbourhoods
    return eng, geom


def _raise_on_status(eng: ForceEngine) -> None:
    if eng.read_status() is not None:
        raise MinimumSeparationError(_MINSEP_MSG)


def _base_mask(eng: ForceEngine, geom: _grid.Geometry, base_cells):
    """Ranks whose cell is one of `base_cells` (the write-discipline view)."""
    cells = np.asarray(base_cells, dtype=np.int64).ravel()
    cor = eng.cell_of_rank[: eng.n].cpu().numpy()
    return np.isin(cor, cells)


def _finish(eng, geom, forces_dev, e_slot, w_slot, base_cells):
    forces = forces_dev.cpu().numpy()
    if base_cells is None:
        sc = eng.scalar_values()
        return forces, float(sc[e_slot]), float(sc[w_slot])
    keep = _base_mask(eng, geom, base_cells)
    parts = eng.parts[: eng.n].cpu().numpy()
    owned = np.zeros(eng.n, dtype=bool)
    owned[parts[keep]] = True
    forces[~owned] = 0.0
    pair = e_slot == SCALAR_E2
    e = (eng.e2_rank if pair else eng.e3_rank)[: eng.n].cpu().numpy()
    w = (eng.w2_rank if pair else eng.w3_rank)[: eng.n].cpu().numpy()
    return forces, float(np.sum(e[keep])), float(np.sum(w[keep]))


def build_cell_grid(system, cutoff: float) -> _grid.CellGrid:
    """GPU binning with the reference's geometry (containers.py:235-279).

    ``cell_start``/``cell_particles`` come from the device counting sort and
    equal the reference's bit for bit; stencil tables are the host restatement.
    """
    eng = engine_for(system.positions.shape[0])
    geom = _geometry_for(system, cutoff)
    eng.upload_positions(system.positions)
    eng.bin(geom)
    pair, patterns, same = _grid.stencil(geom)
    nc = geom.num_cells
    return _grid.CellGrid(
        cells_per_dim=np.array(geom.cells, dtype=np.int64),
        cell_size=np.array(geom.cell_size), origin=np.array(geom.origin),
        interaction_reach=np.array(geom.reach, dtype=np.int64), cutoff=float(cutoff),
        periodic=bool(system.periodic), box=np.asarray(system.box, dtype=np.float64).copy(),
        cell_start=eng.cell_start[: nc + 1].cpu().numpy().astype(np.int64),
        cell_particles=eng.parts[: eng.n].cpu().numpy().astype(np.int64),
        pair_cells=pair.copy(), triplet_patterns=patterns.copy(), triplet_same_cell=same.copy(),
    )


def c01_pair_pass(grid, system, ff, base_cells=None):
    """LJ pass; (forces (n,3), energy, virial) as containers.py:750-783 returns."""
    eng, geom = _prepare(system, grid.cutoff)
    out = eng.torch.empty((eng.n, 3), dtype=eng.torch.float64, device=eng.device)
    eng.lj(geom, grid.cutoff, ff.epsilon, ff.sigma, out, tag=0)
    _raise_on_status(eng)
    return _finish(eng, geom, out, SCALAR_E2, SCALAR_W2, base_cells)


def c01_triplet_pass(grid, system, ff, base_cells=None):
    """ATM pass; (forces (n,3), energy, virial) as containers.py:786-822 returns.

    With ``base_cells`` the C01 (owner-computes) kernel runs, so the energy is
    the reference's per-visit attribution restricted to those cells."""
    if base_cells is not None:
        return c01_triplet_pass_owner(grid, system, ff, base_cells)
    eng, geom = _prepare(system, grid.cutoff)
    out = eng.torch.empty((eng.n, 3), dtype=eng.torch.float64, device=eng.device)
    eng.atm(geom, grid.cutoff, ff.nu, out, tag=0)
    _raise_on_status(eng)
    return _finish(eng, geom, out, SCALAR_E3, SCALAR_W3, base_cells)


def collect_triplet_visits(grid, system, base_cells=None) -> np.ndarray:
    """Sorted (i, j, k) row per accepted visit (containers.py:825-849)."""
    eng, geom = _prepare(system, grid.cutoff)
    out = eng.torch.empty((eng.n, 3), dtype=eng.torch.float64, device=eng.device)
    eng.atm_c01(geom, grid.cutoff, 0.0, out, tag=0)
    rows = eng.visit_rows(geom, grid.cutoff)
    if base_cells is not None:
        parts = eng.parts[: eng.n].cpu().numpy()
        keep = _base_mask(eng, geom, base_cells)
        counts = eng.v_rank[: eng.n].cpu().numpy().astype(np.int64)
        sel = np.repeat(keep, counts)
        rows = rows[sel]
        del parts
    return rows


def triplet_count(system, cutoff: float) -> int:
    """Unique within-cutoff triplets, counted by the Newton-3 enumeration."""
    eng, geom = _prepare(system, cutoff)
    out = eng.torch.empty((eng.n, 3), dtype=eng.torch.float64, device=eng.device)
    eng.atm(geom, cutoff, 0.0, out, tag=0)
    return int(eng.visits.item())


def triplet_visit_count(system, cutoff: float) -> int:
    """Accepted C01 visits (3 per unique triplet), counted by the C01 enumeration."""
    eng, geom = _prepare(system, cutoff)
    out = eng.torch.empty((eng.n, 3), dtype=eng.torch.float64, device=eng.device)
    eng.atm_c01(geom, cutoff, 0.0, out, tag=0)
    return int(eng.visits.item())


def c01_triplet_pass_owner(grid, system, ff, base_cells=None):
    """The same pass through the C01 (owner-computes) kernel, for cross-checks."""
    eng, geom = _prepare(system, grid.cutoff)
    out = eng.torch.empty((eng.n, 3), dtype=eng.torch.float64, device=eng.device)
    eng.atm_c01(geom, grid.cutoff, ff.nu, out, tag=0)
    _raise_on_status(eng)
    return _finish(eng, geom, out, SCALAR_E3, SCALAR_W3, base_cells)


class CudaLinkedCells:
    """GPU drop-in for ``respamd.containers.LinkedCells`` (containers.py:911-937).

    The three-body cutoff is ``ff.cutoff_3b`` when the force field has one
    (this package's ``ForceField``), else ``ff.cutoff`` as in the reference.
    """

    name = "cuda_linked_cells"

    def __init__(self):
        self.pair_energy = 0.0
        self.pair_virial = 0.0
        self.triplet_energy = 0.0
        self.triplet_virial = 0.0
        self.triplet_visits = 0

    @property
    def triplet_count(self) -> int:
        """Unique triplets of the most recent triplet pass."""
        return self.triplet_visits // 3

    def pair_pass(self, system, ff) -> None:
        eng, geom = _prepare(system, ff.cutoff)
        out = eng.torch.empty((eng.n, 3), dtype=eng.torch.float64, device=eng.device)
        eng.lj(geom, ff.cutoff, ff.epsilon, ff.sigma, out, tag=0)
        _raise_on_status(eng)
        forces, e, w = _finish(eng, geom, out, SCALAR_E2, SCALAR_W2, None)
        system.forces_2b[:] = forces
        self.pair_energy, self.pair_virial = e, w

    def triplet_pass(self, system, ff) -> None:
        if ff.nu == 0.0:  # containers.py:928-932
            system.forces_3b[:] = 0.0
            self.triplet_energy = 0.0
            self.triplet_virial = 0.0
            self.triplet_visits = 0
            return
        rc3 = triplet_cutoff(ff)
        eng, geom = _prepare(system, rc3)
        out = eng.torch.empty((eng.n, 3), dtype=eng.torch.float64, device=eng.device)
        eng.atm(geom, rc3, ff.nu, out, tag=0)
        _raise_on_status(eng)
        forces, e, w = _finish(eng, geom, out, SCALAR_E3, SCALAR_W3, None)
        system.forces_3b[:] = forces
        self.triplet_energy, self.triplet_virial = e, w
        self.triplet_visits = 3 * int(eng.visits.item())  # C01-equivalent visit count


# ---------------------------------------------------------------- DirectSum
_DIRECT_PERIODIC_MSG = "DirectSum does not support periodic boundaries"


def _direct_engine(system):
    if system.periodic:  # containers.py:854-855, 866-867
        raise ValidationError(_DIRECT_PERIODIC_MSG)
    eng = engine_for(system.positions.shape[0])
    eng.upload_positions(system.positions)
    eng.reset_status(0)
    return eng


def direct_sum_pairs(system, ff):
    """Every distinct pair, no cutoff (containers.py:852-861); (forces, energy, virial)."""
    eng = _direct_engine(system)
    out = eng.torch.empty((eng.n, 3), dtype=eng.torch.float64, device=eng.device)
    eng.direct_pairs(ff.epsilon, ff.sigma, out, tag=0)
    _raise_on_status(eng)
    sc = eng.scalar_values()
    return out.cpu().numpy(), float(sc[SCALAR_E2]), float(sc[SCALAR_W2])


def direct_sum_triplets(system, ff):
    """Every distinct triplet, no cutoff (containers.py:864-875); (forces, energy, virial)."""
    eng = _direct_engine(system)
    out = eng.torch.empty((eng.n, 3), dtype=eng.torch.float64, device=eng.device)
    eng.direct_triplets(ff.nu, out, tag=0)
    _raise_on_status(eng)
    sc = eng.scalar_values()
    return out.cpu().numpy(), float(sc[SCALAR_E3]), float(sc[SCALAR_W3])


class CudaDirectSum:
    """GPU drop-in for ``respamd.containers.DirectSum`` (containers.py:888-908):
    all pairs and all triplets, no cutoff, non-periodic systems only."""

    name = "cuda_direct_sum"

    def __init__(self):
        self.pair_energy = 0.0
        self.pair_virial = 0.0
        self.triplet_energy = 0.0
        self.triplet_virial = 0.0

    def pair_pass(self, system, ff) -> None:
        forces, self.pair_energy, self.pair_virial = direct_sum_pairs(system, ff)
        system.forces_2b[:] = forces

    def triplet_pass(self, system, ff) -> None:
        if ff.nu == 0.0:  # containers.py:900-904
            system.forces_3b[:] = 0.0
            self.triplet_energy = 0.0
            self.triplet_virial = 0.0
            return
        forces, self.triplet_energy, self.triplet_virial = direct_sum_triplets(system, ff)
        system.forces_3b[:] = forces


def make_container(kind: str):
    """Container factory (containers.py:940-945) for this package's kinds."""
    if kind in ("cuda_linked_cells", "linked_cells"):
        return CudaLinkedCells()
    if kind in ("cuda_direct_sum", "direct_sum"):
        return CudaDirectSum()
    raise ValidationError(f"unknown container kind {kind!r} (this package provides "
                          f"'cuda_linked_cells' and 'cuda_direct_sum')")
