"""CPU oracle for the force-evaluation hot path -- TEST INFRASTRUCTURE ONLY.

This module is the checker, never the product.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and
``--impl reference`` arm) may import it.  The product package
``paper_2507_11172_b200`` never imports, links or calls anything here.

It restates the reference package ``respamd`` (``/root/reference/pkg/src``)
for the hot path:

* numeric kernels -> ``oracle.c`` (ctypes, built by ``oracle/Makefile``);
* host-side stencil tables, grid geometry, pass wrappers, the r-RESPA loop
  and ``wrap_positions`` -> numpy below, each citing the reference line it
  follows.

Parity of the restatement with the live reference is pinned by
``tests/golden/*.npz`` (made by ``tests/golden/make_golden.py``, which runs
the reference itself) and checked in ``tests/test_oracle_golden.py``.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

MIN_DISTANCE_SQ = 1e-10 * 1e-10  # respamd/potentials.py:35-36


class OracleValidationError(ValueError):
    """Mirror of respamd.model.ValidationError (model.py:16-17)."""


class OracleMinimumSeparationError(OracleValidationError):
    """Mirror of respamd.containers.MinimumSeparationError (containers.py:39-40)."""


class OracleBlowUp(RuntimeError):
    """Mirror of respamd.integrators.IntegrationBlowUp (integrators.py:29-35)."""

    def __init__(self, iteration, reason, trace=None):
        self.iteration = iteration
        self.trace = trace
        super().__init__(f"integration blew up at iteration {iteration}: {reason}")


def build(force: bool = False) -> str:
    """Compile oracle.c into liboracle.so (make)."""
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(
        os.path.join(_HERE, "oracle.c")
    ):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB_PATH)
        P = ctypes.c_void_p
        I64 = ctypes.c_int64
        D = ctypes.c_double
        L.orc_lj_kernel.argtypes = [D, D, D, P]
        L.orc_atm_kernel.argtypes = [D, D, D, D, P]
        L.orc_bin_particles.argtypes = [I64, P, P, P, P, P, P]
        L.orc_c01_pair.argtypes = [P, P, ctypes.c_int, P, P, P, P, I64, D, D, D, P, I64, P, P, P, P]
        L.orc_c01_triplet.argtypes = [
            P, P, ctypes.c_int, P, P, P, P, I64, P, P, I64, D, D, P, I64, P, P, P, P,
        ]
        L.orc_c01_triplet_visit_counts.argtypes = [
            P, P, ctypes.c_int, P, P, P, P, I64, P, P, I64, D, P, I64, P,
        ]
        L.orc_brute_pairs.argtypes = [I64, P, P, ctypes.c_int, D, D, D, P, P]
        L.orc_brute_triplets.argtypes = [I64, P, P, ctypes.c_int, D, D, P, P]
        L.orc_brute_triplets.restype = I64
        L.orc_direct_pairs.argtypes = [I64, P, D, D, I64, P, P, P, P]
        L.orc_direct_triplets.argtypes = [I64, P, D, I64, P, P, P, P]
        L.orc_distance_histogram.argtypes = [I64, P, P, D, I64, P]
        L.orc_set_num_threads.argtypes = [ctypes.c_int]
        L.orc_get_max_threads.restype = ctypes.c_int
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def set_num_threads(n: int) -> None:
    lib().orc_set_num_threads(int(n))


def get_max_threads() -> int:
    return int(lib().orc_get_max_threads())


# ---------------------------------------------------------------------------
# scalar kernels
# ---------------------------------------------------------------------------


def lj_kernel(r2, epsilon, sigma2):
    """respamd/potentials.py:55-67."""
    out = np.zeros(2)
    lib().orc_lj_kernel(float(r2), float(epsilon), float(sigma2), _p(out))
    return float(out[0]), float(out[1])


def atm_kernel(a, b, c, nu):
    """respamd/potentials.py:82-114."""
    out = np.zeros(4)
    lib().orc_atm_kernel(float(a), float(b), float(c), float(nu), _p(out))
    return tuple(float(v) for v in out)


# ---------------------------------------------------------------------------
# grid geometry and stencil tables (host side, numpy/python)
# ---------------------------------------------------------------------------


def _cell_gap_distance(delta, cells_per_dim, cell_size, periodic) -> float:
    """respamd/containers.py:75-86."""
    d2 = 0.0
    for d in range(3):
        dd = abs(int(delta[d]))
        if periodic:
            n = int(cells_per_dim[d])
            dd = dd % n
            dd = min(dd, n - dd)
        gap = max(0, dd - 1) * float(cell_size[d])
        d2 += gap * gap
    return float(np.sqrt(d2))


def _offset_cube(reach):
    """respamd/containers.py:89-97."""
    rx, ry, rz = (int(r) for r in reach)
    return [(x, y, z) for x in range(-rx, rx + 1) for y in range(-ry, ry + 1) for z in range(-rz, rz + 1)]


def stencil_tables(cells, size, reach, cutoff, periodic):
    """Canonical pair offsets and triplet patterns.

    Restates generate_pair_offsets (containers.py:100-109),
    generate_triplet_offsets (:112-130), _canonical_pair_offsets (:133-144)
    and _canonical_triplet_offsets (:147-172).
    """
    cube = _offset_cube(reach)
    reachable = [o for o in cube if _cell_gap_distance(o, cells, size, periodic) <= cutoff]
    pair = np.array(reachable, dtype=np.int64).reshape(-1, 3)
    if periodic:
        pair = np.unique(np.mod(pair, np.asarray(cells)[None, :]), axis=0)
    index_of = {tuple(int(v) for v in row): idx for idx, row in enumerate(pair)}

    def canonical(o):
        if periodic:
            return tuple(int(v) % int(n) for v, n in zip(o, cells))
        return tuple(int(v) for v in o)

    pairs = set()
    for c1 in reachable:
        for c2 in reachable:
            if tuple(c1) > tuple(c2):
                continue
            delta = tuple(b - a for a, b in zip(c1, c2))
            if _cell_gap_distance(delta, cells, size, periodic) <= cutoff:
                i1, i2 = index_of[canonical(c1)], index_of[canonical(c2)]
                pairs.add((min(i1, i2), max(i1, i2)))
    rows = np.array(sorted(pairs), dtype=np.int64).reshape(-1, 2)
    same = rows[:, 0] == rows[:, 1]
    return pair, rows, same


@dataclass
class OracleGrid:
    """Restatement of respamd.containers.CellGrid (containers.py:50-72)."""

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


def grid_geometry(box, positions, cutoff, periodic):
    """(origin, extent, cells, size, reach) as containers.py:244-262 computes them."""
    box = np.asarray(box, dtype=np.float64)
    if cutoff <= 0:
        raise OracleValidationError(f"cutoff must be > 0, got {cutoff}")
    if periodic:
        if np.any(box < 2.0 * cutoff):
            raise OracleValidationError("periodic box too small for minimum-image safety")
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
    return origin, extent, cells, size, reach


def bin_particles(positions, origin, inv_cell, cells):
    """respamd/containers.py:175-209 via orc_bin_particles."""
    positions = np.ascontiguousarray(positions, dtype=np.float64)
    origin = np.ascontiguousarray(origin, dtype=np.float64)
    inv_cell = np.ascontiguousarray(inv_cell, dtype=np.float64)
    cells = np.ascontiguousarray(cells, dtype=np.int64)
    n = positions.shape[0]
    start = np.zeros(int(np.prod(cells)) + 1, np.int64)
    parts = np.zeros(n, np.int64)
    lib().orc_bin_particles(n, _p(positions), _p(origin), _p(inv_cell), _p(cells), _p(start), _p(parts))
    return start, parts


def build_cell_grid(system, cutoff) -> OracleGrid:
    """respamd/containers.py:235-279."""
    origin, _, cells, size, reach = grid_geometry(system.box, system.positions, cutoff, system.periodic)
    start, parts = bin_particles(system.positions, origin, 1.0 / size, cells)
    pair, patterns, same = stencil_tables(cells, size, reach, float(cutoff), system.periodic)
    return OracleGrid(
        cells_per_dim=cells,
        cell_size=size,
        origin=origin,
        interaction_reach=reach,
        cutoff=float(cutoff),
        periodic=bool(system.periodic),
        box=np.asarray(system.box, dtype=np.float64).copy(),
        cell_start=start,
        cell_particles=parts,
        pair_cells=np.ascontiguousarray(pair),
        triplet_patterns=np.ascontiguousarray(patterns),
        triplet_same_cell=np.ascontiguousarray(same),
    )


def _check_flags(flags):
    """respamd/containers.py:742-747."""
    if np.any(flags):
        raise OracleMinimumSeparationError("particles closer than the minimum separation guard")


def _base(grid, base_cells):
    if base_cells is None:
        return np.arange(grid.num_cells, dtype=np.int64)
    return np.ascontiguousarray(base_cells, dtype=np.int64)


def c01_pair_pass(grid: OracleGrid, system, ff, base_cells=None, cutoff=None):
    """respamd/containers.py:750-783; returns (forces, energy, virial)."""
    pos = np.ascontiguousarray(system.positions, dtype=np.float64)
    rc = grid.cutoff if cutoff is None else float(cutoff)
    base = _base(grid, base_cells)
    forces = np.zeros((pos.shape[0], 3))
    ce = np.zeros(grid.num_cells)
    cw = np.zeros(grid.num_cells)
    flags = np.zeros(grid.num_cells, np.int64)
    lib().orc_c01_pair(
        _p(pos), _p(grid.box), int(grid.periodic), _p(grid.cells_per_dim), _p(grid.cell_start),
        _p(grid.cell_particles), _p(grid.pair_cells), grid.pair_cells.shape[0], rc * rc,
        float(ff.epsilon), float(ff.sigma) * float(ff.sigma), _p(base), base.shape[0], _p(forces),
        _p(ce), _p(cw), _p(flags),
    )
    _check_flags(flags)
    return forces, float(np.sum(ce)), float(np.sum(cw))


def c01_triplet_pass(grid: OracleGrid, system, ff, base_cells=None):
    """respamd/containers.py:786-822; returns (forces, energy, virial)."""
    pos = np.ascontiguousarray(system.positions, dtype=np.float64)
    base = _base(grid, base_cells)
    same = grid.triplet_same_cell.astype(np.uint8)
    forces = np.zeros((pos.shape[0], 3))
    ce = np.zeros(grid.num_cells)
    cw = np.zeros(grid.num_cells)
    flags = np.zeros(grid.num_cells, np.int64)
    lib().orc_c01_triplet(
        _p(pos), _p(grid.box), int(grid.periodic), _p(grid.cells_per_dim), _p(grid.cell_start),
        _p(grid.cell_particles), _p(grid.pair_cells), grid.pair_cells.shape[0],
        _p(grid.triplet_patterns), _p(same), grid.triplet_patterns.shape[0],
        grid.cutoff * grid.cutoff, float(ff.nu), _p(base), base.shape[0], _p(forces), _p(ce), _p(cw),
        _p(flags),
    )
    _check_flags(flags)
    return forces, float(np.sum(ce)), float(np.sum(cw))


def triplet_visit_count(grid: OracleGrid, system, base_cells=None) -> int:
    """Number of rows collect_triplet_visits (containers.py:825-849) returns."""
    pos = np.ascontiguousarray(system.positions, dtype=np.float64)
    base = _base(grid, base_cells)
    same = grid.triplet_same_cell.astype(np.uint8)
    visits = np.zeros(grid.num_cells, np.int64)
    lib().orc_c01_triplet_visit_counts(
        _p(pos), _p(grid.box), int(grid.periodic), _p(grid.cells_per_dim), _p(grid.cell_start),
        _p(grid.cell_particles), _p(grid.pair_cells), grid.pair_cells.shape[0],
        _p(grid.triplet_patterns), _p(same), grid.triplet_patterns.shape[0],
        grid.cutoff * grid.cutoff, _p(base), base.shape[0], _p(visits),
    )
    return int(visits.sum())


def brute_force_pairs(system, ff, cutoff=None):
    """respamd/reference.py:111-115 -> (forces, energy, virial)."""
    pos = np.ascontiguousarray(system.positions, dtype=np.float64)
    rc2 = np.inf if cutoff is None else float(cutoff) ** 2
    forces = np.zeros_like(pos)
    out = np.zeros(2)
    box = np.ascontiguousarray(system.box, dtype=np.float64)
    lib().orc_brute_pairs(
        pos.shape[0], _p(pos), _p(box), int(system.periodic), rc2, float(ff.epsilon),
        float(ff.sigma) ** 2, _p(forces), _p(out),
    )
    return forces, float(out[0]), float(out[1])


def brute_force_triplets(system, ff, cutoff=None):
    """respamd/reference.py:118-122 -> (forces, energy, virial, count)."""
    pos = np.ascontiguousarray(system.positions, dtype=np.float64)
    rc2 = np.inf if cutoff is None else float(cutoff) ** 2
    forces = np.zeros_like(pos)
    out = np.zeros(2)
    box = np.ascontiguousarray(system.box, dtype=np.float64)
    count = lib().orc_brute_triplets(
        pos.shape[0], _p(pos), _p(box), int(system.periodic), rc2, float(ff.nu), _p(forces), _p(out)
    )
    return forces, float(out[0]), float(out[1]), int(count)


# ---------------------------------------------------------------------------
# container + integrator restatement
# ---------------------------------------------------------------------------


def distance_histogram(positions, box, r_max, bins) -> np.ndarray:
    """respamd/observables.py:143-177 -> int64 counts (2 per unordered pair)."""
    pos = np.ascontiguousarray(positions, dtype=np.float64)
    box = np.ascontiguousarray(box, dtype=np.float64)
    counts = np.zeros(int(bins), np.int64)
    lib().orc_distance_histogram(pos.shape[0], _p(pos), _p(box), float(r_max), int(bins),
                                 _p(counts))
    return counts


DIRECT_SUM_CHUNKS = 16  # respamd/containers.py:36


def _direct_buffers(n):
    return (np.zeros((DIRECT_SUM_CHUNKS, n, 3)), np.zeros(DIRECT_SUM_CHUNKS),
            np.zeros(DIRECT_SUM_CHUNKS), np.zeros(DIRECT_SUM_CHUNKS, np.int64))


def direct_sum_pairs(system, ff):
    """respamd/containers.py:852-861 (kernel :663-692) -> (forces, energy, virial)."""
    if system.periodic:
        raise OracleValidationError("DirectSum does not support periodic boundaries")
    pos = np.ascontiguousarray(system.positions, dtype=np.float64)
    fbuf, ebuf, wbuf, flags = _direct_buffers(pos.shape[0])
    lib().orc_direct_pairs(pos.shape[0], _p(pos), float(ff.epsilon), float(ff.sigma) ** 2,
                           DIRECT_SUM_CHUNKS, _p(fbuf), _p(ebuf), _p(wbuf), _p(flags))
    _check_flags(flags)
    return fbuf.sum(axis=0), float(np.sum(ebuf)), float(np.sum(wbuf))


def direct_sum_triplets(system, ff):
    """respamd/containers.py:864-875 (kernel :695-739) -> (forces, energy, virial)."""
    if system.periodic:
        raise OracleValidationError("DirectSum does not support periodic boundaries")
    pos = np.ascontiguousarray(system.positions, dtype=np.float64)
    fbuf, ebuf, wbuf, flags = _direct_buffers(pos.shape[0])
    lib().orc_direct_triplets(pos.shape[0], _p(pos), float(ff.nu), DIRECT_SUM_CHUNKS, _p(fbuf),
                              _p(ebuf), _p(wbuf), _p(flags))
    _check_flags(flags)
    return fbuf.sum(axis=0), float(np.sum(ebuf)), float(np.sum(wbuf))


class OracleDirectSum:
    """respamd/containers.py:888-908."""

    name = "direct_sum"

    def __init__(self):
        self.pair_energy = self.pair_virial = 0.0
        self.triplet_energy = self.triplet_virial = 0.0

    def pair_pass(self, system, ff):
        f, self.pair_energy, self.pair_virial = direct_sum_pairs(system, ff)
        system.forces_2b[:] = f

    def triplet_pass(self, system, ff):
        if ff.nu == 0.0:
            system.forces_3b[:] = 0.0
            self.triplet_energy = self.triplet_virial = 0.0
            return
        f, self.triplet_energy, self.triplet_virial = direct_sum_triplets(system, ff)
        system.forces_3b[:] = f


class OracleLinkedCells:
    """respamd.containers.LinkedCells (containers.py:911-937), with an
    optional separate three-body cutoff (the split-cutoff adapter of
    SURVEY.md §7 step 1; rc3=None keeps the reference's single cutoff)."""

    name = "linked_cells"

    def __init__(self, rc3=None):
        self.rc3 = rc3
        self.pair_energy = 0.0
        self.pair_virial = 0.0
        self.triplet_energy = 0.0
        self.triplet_virial = 0.0
        self.triplet_visits = 0

    def pair_pass(self, system, ff) -> None:
        grid = build_cell_grid(system, ff.cutoff)
        forces, e, w = c01_pair_pass(grid, system, ff)
        system.forces_2b[:] = forces
        self.pair_energy, self.pair_virial = e, w

    def triplet_pass(self, system, ff) -> None:
        if ff.nu == 0.0:
            system.forces_3b[:] = 0.0
            self.triplet_energy = 0.0
            self.triplet_virial = 0.0
            return
        rc = ff.cutoff if self.rc3 is None else self.rc3
        grid = build_cell_grid(system, rc)
        forces, e, w = c01_triplet_pass(grid, system, ff)
        system.forces_3b[:] = forces
        self.triplet_energy, self.triplet_virial = e, w


def wrap_positions(positions: np.ndarray, box: np.ndarray) -> None:
    """respamd/model.py:274-280."""
    np.mod(positions, box, out=positions)
    oob = positions >= box
    if np.any(oob):
        positions[oob] = 0.0


@dataclass
class OracleTrace:
    """respamd.integrators.RunTrace (integrators.py:63-86)."""

    iterations: list = field(default_factory=list)
    kinetic: list = field(default_factory=list)
    potential_2b: list = field(default_factory=list)
    potential_3b: list = field(default_factory=list)
    total: list = field(default_factory=list)
    virial_2b: list = field(default_factory=list)
    virial_3b: list = field(default_factory=list)

    def record(self, iteration, system, container):
        kin = 0.5 * system.mass * float(np.sum(system.velocities * system.velocities))
        self.iterations.append(iteration)
        self.kinetic.append(kin)
        self.potential_2b.append(container.pair_energy)
        self.potential_3b.append(container.triplet_energy)
        self.total.append(kin + container.pair_energy + container.triplet_energy)
        self.virial_2b.append(container.pair_virial)
        self.virial_3b.append(container.triplet_virial)


def respa_run(system, ff, container, dt, step_size_factor, num_iterations, sample_interval=None):
    """numpy restatement of respamd.integrators.respa_run (integrators.py:96-173)."""
    s = int(step_size_factor)
    if num_iterations % s != 0:
        raise OracleValidationError("num_iterations must be a multiple of the step_size_factor")
    if sample_interval is None:
        sample_interval = s
    if sample_interval < 1 or sample_interval % s != 0:
        raise OracleValidationError("sample_interval must be a positive multiple of s")
    m = system.mass
    half_dt = 0.5 * dt / m
    half_drift = 0.5 * dt * dt / m
    half_respa = 0.5 * dt * s / m
    trace = OracleTrace()
    try:
        container.pair_pass(system, ff)
        container.triplet_pass(system, ff)
    except OracleMinimumSeparationError as exc:
        raise OracleBlowUp(0, str(exc), trace) from exc
    trace.record(0, system, container)
    f2_old = system.forces_2b.copy()
    for i in range(num_iterations):
        if i % s == 0:
            system.velocities += half_respa * system.forces_3b
        system.positions += dt * system.velocities + half_drift * f2_old
        if system.periodic:
            wrap_positions(system.positions, system.box)
        try:
            container.pair_pass(system, ff)
        except OracleMinimumSeparationError as exc:
            raise OracleBlowUp(i + 1, str(exc), trace) from exc
        system.velocities += half_dt * (f2_old + system.forces_2b)
        np.copyto(f2_old, system.forces_2b)
        if (i + 1) % s == 0:
            try:
                container.triplet_pass(system, ff)
            except OracleMinimumSeparationError as exc:
                raise OracleBlowUp(i + 1, str(exc), trace) from exc
            system.velocities += half_respa * system.forces_3b
        if not (np.all(np.isfinite(system.positions)) and np.all(np.isfinite(system.velocities))):
            raise OracleBlowUp(i + 1, "non-finite state", trace)
        if (i + 1) % sample_interval == 0:
            trace.record(i + 1, system, container)
    return trace


# ---------------------------------------------------------------------------
# a tiny stand-in for respamd.model.ParticleSystem / ForceField
# ---------------------------------------------------------------------------


@dataclass
class OracleSystem:
    positions: np.ndarray
    velocities: np.ndarray
    forces_2b: np.ndarray
    forces_3b: np.ndarray
    mass: float
    box: np.ndarray
    periodic: bool

    @classmethod
    def from_positions(cls, positions, box, periodic=True, velocities=None, mass=1.0):
        positions = np.ascontiguousarray(positions, dtype=np.float64).copy()
        n = positions.shape[0]
        v = np.zeros((n, 3)) if velocities is None else np.ascontiguousarray(velocities, np.float64).copy()
        return cls(positions, v, np.zeros((n, 3)), np.zeros((n, 3)), float(mass),
                   np.asarray(box, dtype=np.float64).copy(), bool(periodic))

    @property
    def n(self):
        return self.positions.shape[0]

    def copy(self):
        return OracleSystem(self.positions.copy(), self.velocities.copy(), self.forces_2b.copy(),
                            self.forces_3b.copy(), self.mass, self.box.copy(), self.periodic)


@dataclass
class OracleForceField:
    epsilon: float = 1.0
    sigma: float = 1.0
    nu: float = 0.0
    cutoff: float = 2.5


def unique_triplet_count(system, cutoff) -> int:
    """Unique within-cutoff triplets = C01 visits / 3 (containers.py:786-795)."""
    grid = build_cell_grid(system, cutoff)
    visits = triplet_visit_count(grid, system)
    assert visits % 3 == 0
    return visits // 3


