"""GPU parity: the sm_100a path against the reference (golden fixtures made by
the reference itself) and against the bit-pinned CPU oracle.

Tolerances (north star / SURVEY.md Appendix A.5):
* cell tables, triplet counts, visit multisets: bit-exact;
* forces: normwise max_i|dF_i| / max_i|F_i| <= 1e-10;
* energies <= 1e-10 relative, virials <= 1e-9 relative (test_containers.py:153);
* trajectories (respa_run): positions/velocities <= 1e-10 absolute.
"""

import glob
import os
from collections import Counter

import numpy as np
import pytest

from helpers import GOLDEN, TEST_SEED, load_golden, normwise, random_positions

pytestmark = pytest.mark.gpu

SMALL = sorted(os.path.basename(p) for p in glob.glob(os.path.join(GOLDEN, "small_*.npz")))
FORCE_TOL = 1e-10
ENERGY_TOL = 1e-10
VIRIAL_TOL = 1e-9


@pytest.fixture(scope="module")
def pkg():
    import paper_2507_11172_b200 as p
    from paper_2507_11172_b200 import _lib

    _lib.require_device()
    return p


def _rel(a, b):
    return abs(a - b) / max(1.0, abs(b))


def _system(pkg, pos, box, periodic, vel=None):
    s = pkg.ParticleSystem.empty(len(pos), box, periodic=periodic)
    s.positions[:] = pos
    if vel is not None:
        s.velocities[:] = vel
    return s


# --------------------------------------------------------------------------
# binning, passes, counts on the small reference fixtures
# --------------------------------------------------------------------------
@pytest.mark.parametrize("name", SMALL)
def test_binning_bit_exact(pkg, name):
    g = load_golden(name)
    s = _system(pkg, g["positions"], g["box"], bool(g["periodic"]))
    grid = pkg.build_cell_grid(s, float(g["cutoff"]))
    assert np.array_equal(grid.cell_start, g["cell_start"])
    assert np.array_equal(grid.cell_particles, g["cell_particles"])
    assert np.array_equal(grid.triplet_patterns, g["triplet_patterns"])


@pytest.mark.parametrize("name", SMALL)
def test_pair_pass_matches_reference(pkg, name):
    g = load_golden(name)
    s = _system(pkg, g["positions"], g["box"], bool(g["periodic"]))
    ff = pkg.ForceField(nu=float(g["nu"]), cutoff=float(g["cutoff"]))
    grid = pkg.build_cell_grid(s, ff.cutoff)
    f, e, w = pkg.c01_pair_pass(grid, s, ff)
    assert normwise(f, g["f2"]) <= FORCE_TOL
    assert np.max(np.abs(f - g["bf2"])) <= 1e-10  # the reference's own C01-vs-brute bound
    assert _rel(e, float(g["e2"])) <= ENERGY_TOL
    assert _rel(w, float(g["w2"])) <= VIRIAL_TOL


@pytest.mark.parametrize("name", SMALL)
def test_triplet_pass_matches_reference(pkg, name):
    g = load_golden(name)
    s = _system(pkg, g["positions"], g["box"], bool(g["periodic"]))
    ff = pkg.ForceField(nu=float(g["nu"]), cutoff=float(g["cutoff"]))
    grid = pkg.build_cell_grid(s, ff.cutoff)
    f, e, w = pkg.c01_triplet_pass(grid, s, ff)
    assert normwise(f, g["f3"]) <= FORCE_TOL
    assert np.max(np.abs(f - g["bf3"])) <= 1e-9
    assert _rel(e, float(g["e3"])) <= ENERGY_TOL
    assert _rel(w, float(g["w3"])) <= VIRIAL_TOL


@pytest.mark.parametrize("name", SMALL)
def test_triplet_visits_bit_exact(pkg, name):
    """Each triplet visited exactly 3x; distinct set == the reference's."""
    g = load_golden(name)
    s = _system(pkg, g["positions"], g["box"], bool(g["periodic"]))
    grid = pkg.build_cell_grid(s, float(g["cutoff"]))
    rows = pkg.collect_triplet_visits(grid, s)
    assert rows.shape[0] == int(g["visits"])
    visits = Counter(map(tuple, rows))
    assert all(v == 3 for v in visits.values())
    ref = {tuple(r) for r in g["unique_triplets"]}
    assert set(visits) == ref
    assert pkg.triplet_count(s, float(g["cutoff"])) == int(g["brute_count"])


@pytest.mark.parametrize("name", SMALL)
def test_newton3_matches_c01_enumeration(pkg, name):
    """The Newton-3 pass (each triplet once) and the C01 pass (each triplet
    from every member) are independent enumerations: same forces, energies
    and counts (unique x 3 == visits)."""
    from paper_2507_11172_b200 import containers as pc

    g = load_golden(name)
    s = _system(pkg, g["positions"], g["box"], bool(g["periodic"]))
    ff = pkg.ForceField(nu=float(g["nu"]), cutoff=float(g["cutoff"]))
    grid = pkg.build_cell_grid(s, ff.cutoff)
    f3, e3, w3 = pkg.c01_triplet_pass(grid, s, ff)
    f1, e1, w1 = pc.c01_triplet_pass_owner(grid, s, ff)
    assert normwise(f3, f1) <= FORCE_TOL
    assert _rel(e3, e1) <= ENERGY_TOL and _rel(w3, w1) <= VIRIAL_TOL
    assert 3 * pkg.triplet_count(s, ff.cutoff) == pc.triplet_visit_count(s, ff.cutoff)


def test_newton3_forces_sum_to_zero(pkg):
    s = pkg.systems.fcc_system(6, jitter=0.05, seed=4)
    ff = pkg.ForceField(nu=0.073, cutoff=2.5)
    c = pkg.CudaLinkedCells()
    c.triplet_pass(s, ff)
    assert np.max(np.abs(s.forces_3b.sum(axis=0))) <= 1e-12 * s.n


@pytest.mark.parametrize("nc,r_list", [(10, 2.8), (6, 3.4), (4, 2.6)])
def test_fused_rebuild_equals_separate_kernels(pkg, nc, r_list):
    """rb_rebuild (one launch, grid barriers) writes exactly what rb_bin +
    rb_nlist + rb_nlist_mirror write; with the gate closed it writes nothing."""
    import torch

    from paper_2507_11172_b200.engine import ForceEngine
    from paper_2507_11172_b200.grid import geometry

    s = pkg.systems.fcc_system(nc, jitter=0.05, seed=nc)
    n = s.positions.shape[0]
    geom = geometry(s.box, None, r_list, True)
    a, b = ForceEngine(n), ForceEngine(n)
    for e in (a, b):
        e.upload_positions(s.positions)
    a.bin(geom)
    a.nlist(geom, r_list, checked=True)
    b.rebuild(geom, r_list, a.capacity, tag=0, fused=True)  # flag 0 == tag 0: open
    ncell = geom.num_cells
    for name, k in (("cell_start", ncell + 1), ("parts", n), ("cell_of_rank", n),
                    ("rank_of", n), ("row_count", n)):
        assert np.array_equal(getattr(a, name)[:k].cpu().numpy(),
                              getattr(b, name)[:k].cpu().numpy()), name
    for name in ("pos_r", "x_ref"):
        assert np.array_equal(getattr(a, name)[:n].cpu().numpy(),
                              getattr(b, name)[:n].cpu().numpy()), name
    cnt = a.row_count[:n].cpu().numpy()
    cap = a.capacity
    ra, rb_ = (e.rows[:n * cap].cpu().numpy().reshape(n, cap) for e in (a, b))
    ma, mb = (e.mirror[:n * cap].cpu().numpy().reshape(n, cap) for e in (a, b))
    valid = np.arange(cap)[None, :] < cnt[:, None]
    assert np.array_equal(ra[valid], rb_[valid])
    # mirror: the entries above the diagonal (the ones the header defines),
    # each the position of p in row q
    upper = valid & (ra > np.arange(n)[:, None])
    assert np.array_equal(ma[upper], mb[upper])
    p_idx, k_idx = np.nonzero(upper)
    q_idx = ra[p_idx, k_idx]
    assert np.array_equal(ra[q_idx, ma[p_idx, k_idx]], p_idx)
    assert int(a.max_count.item()) == int(b.max_count.item())
    # gate closed (flag != tag): nothing is written
    before = b.rows.clone()
    b.upload_positions(s.positions[::-1].copy())
    b.rebuild(geom, r_list, a.capacity, tag=5, fused=True)
    assert torch.equal(before, b.rows)


def test_write_discipline_single_base_cell(pkg, rng):
    pos = random_positions(rng, 150, (10.0,) * 3, True)
    s = _system(pkg, pos, (10.0,) * 3, True)
    ff = pkg.ForceField(nu=0.7, cutoff=2.5)
    grid = pkg.build_cell_grid(s, ff.cutoff)
    base = int(np.argmax(np.diff(grid.cell_start)))
    owned = set(grid.particles_of_cell(base).tolist())
    for fn in (pkg.c01_pair_pass, pkg.c01_triplet_pass):
        f, _, _ = fn(grid, s, ff, base_cells=[base])
        touched = {int(i) for i in np.nonzero(np.any(f != 0.0, axis=1))[0]}
        assert touched <= owned and touched


def test_closed_forms(pkg):
    """test_containers.py:109-143: LJ minimum and equilateral ATM triangle."""
    ff = pkg.ForceField(nu=0.7, cutoff=2.5)
    r = 2.0 ** (1.0 / 6.0)
    s = _system(pkg, np.array([[1.0, 1.0, 1.0], [1.0 + r, 1.0, 1.0]]), (10.0,) * 3, True)
    f, e, _ = pkg.c01_pair_pass(pkg.build_cell_grid(s, 2.5), s, ff)
    assert np.max(np.abs(f)) < 1e-12 and abs(e + 1.0) < 1e-12
    r = 1.2
    pts = np.array([[1.0, 1.0, 1.0], [1.0 + r, 1.0, 1.0], [1.0 + r / 2, 1.0 + r * np.sqrt(3) / 2, 1.0]])
    s = _system(pkg, pts, (10.0,) * 3, True)
    f, e, _ = pkg.c01_triplet_pass(pkg.build_cell_grid(s, 2.5), s, ff)
    assert abs(e - 1.375 * 0.7 / r ** 9) <= 1e-12 * abs(e)
    assert np.max(np.abs(f.sum(axis=0))) < 1e-12
    s1 = _system(pkg, np.array([[2.5, 2.5, 2.5]]), (10.0,) * 3, True)
    f, e, w = pkg.c01_pair_pass(pkg.build_cell_grid(s1, 2.5), s1, ff)
    assert np.all(f == 0.0) and e == 0.0 and w == 0.0


def test_random_systems_against_oracle(pkg, oracle, rng):
    """Acceptance-style sweep (test_acceptance.py:114-150): 30 random periodic
    systems, GPU vs the oracle's brute-force enumeration."""
    ff = pkg.ForceField(nu=0.6, cutoff=2.5)
    off = oracle.OracleForceField(nu=0.6, cutoff=2.5)
    for _ in range(30):
        edge = rng.uniform(6.0, 10.0)
        n = min(200, int(rng.uniform(0.3, 0.6) * edge ** 3))
        pos = random_positions(rng, n, (edge,) * 3, True, min_sep=0.8)
        s = _system(pkg, pos, (edge,) * 3, True)
        grid = pkg.build_cell_grid(s, 2.5)
        f2, e2, _ = pkg.c01_pair_pass(grid, s, ff)
        f3, e3, _ = pkg.c01_triplet_pass(grid, s, ff)
        os_ = oracle.OracleSystem.from_positions(pos, (edge,) * 3, True)
        rf2, re2, _ = oracle.brute_force_pairs(os_, off, cutoff=2.5)
        rf3, re3, _, count = oracle.brute_force_triplets(os_, off, cutoff=2.5)
        assert np.max(np.abs(f2 - rf2)) <= 1e-9 and np.max(np.abs(f3 - rf3)) <= 1e-9
        assert _rel(e2, re2) <= 1e-10 and _rel(e3, re3) <= 1e-10
        assert pkg.triplet_count(s, 2.5) == count


def test_triplet_overflow_launch_matches_oracle(pkg, oracle, monkeypatch):
    """Bases whose S+ exceeds the main launch's slots go to the second
    (full-slot) launch of the row-based pass; the forces must not depend on
    which launch ran."""
    from paper_2507_11172_b200.containers import engine_for
    from paper_2507_11172_b200.engine import ForceEngine

    monkeypatch.setattr(ForceEngine, "CELLS_MODE", "0")  # the row-based pass

    s = pkg.systems.fcc_system(9, jitter=0.05, seed=9)  # rows of ~130: 160 slots, split
    ff = pkg.ForceField(nu=0.4, cutoff=3.4)
    c = pkg.CudaLinkedCells()
    c.triplet_pass(s, ff)
    eng = engine_for(s.positions.shape[0])
    assert eng.slots > 128
    import torch

    words = eng.atm_scratch.view(torch.int32)  # base counter, count, diagnostic, list, ...
    listed = int(words[2].item())  # the last pass's overflow count
    assert 0 < listed < eng.n
    os_ = oracle.OracleSystem.from_positions(s.positions, s.box, True)
    off = oracle.OracleForceField(nu=0.4, cutoff=3.4)
    rf3, re3, _, count = oracle.brute_force_triplets(os_, off, cutoff=3.4)
    assert normwise(s.forces_3b, rf3) <= FORCE_TOL
    assert _rel(c.triplet_energy, re3) <= ENERGY_TOL
    assert c.triplet_count == count


def test_open_boundaries_against_oracle(pkg, oracle, rng):
    """Non-periodic grids (origin/extent from the particles, containers.py:255-259)."""
    ff = pkg.ForceField(nu=0.7, cutoff=2.5)
    off = oracle.OracleForceField(nu=0.7, cutoff=2.5)
    for n, edge in ((40, 6.0), (90, 7.5)):
        pos = random_positions(rng, n, (edge,) * 3, False)
        pos[0] += 0.7 * edge  # drifted outside the box
        s = _system(pkg, pos, (edge,) * 3, False)
        grid = pkg.build_cell_grid(s, 2.5)
        f2, e2, _ = pkg.c01_pair_pass(grid, s, ff)
        f3, e3, _ = pkg.c01_triplet_pass(grid, s, ff)
        os_ = oracle.OracleSystem.from_positions(pos, (edge,) * 3, False)
        ogrid = oracle.build_cell_grid(os_, 2.5)
        assert np.array_equal(grid.cell_particles, ogrid.cell_particles)
        rf2, re2, _ = oracle.brute_force_pairs(os_, off, cutoff=2.5)
        rf3, re3, _, count = oracle.brute_force_triplets(os_, off, cutoff=2.5)
        assert np.max(np.abs(f2 - rf2)) <= 1e-9 and np.max(np.abs(f3 - rf3)) <= 1e-9
        assert _rel(e3, re3) <= 1e-10
        assert pkg.triplet_count(s, 2.5) == count


def test_minimum_separation_raises(pkg):
    ff = pkg.ForceField(nu=0.7, cutoff=2.5)
    s = _system(pkg, np.array([[1.0, 1.0, 1.0], [1.0 + 5e-11, 1.0, 1.0], [2.0, 1.0, 1.0]]),
                (10.0,) * 3, True)
    c = pkg.CudaLinkedCells()
    with pytest.raises(pkg.MinimumSeparationError):
        c.pair_pass(s, ff)
    with pytest.raises(pkg.MinimumSeparationError):
        c.triplet_pass(s, ff)


def test_minimum_separation_between_slots_raises(pkg, rng):
    """The guard on r_jk (potentials.py:35-36) inside the register-resident
    rounds: two slots of a lower-ranked base almost coincide, so the fp64
    estimate a + b - 2 g of r_jk^2 rounds to ~0 (either sign); the pair is
    settled by the reference arithmetic and the pass raises, as the
    reference does -- for a bare triplet and inside a liquid-density box."""
    ff = pkg.ForceField(nu=0.7, cutoff=2.5)
    c = pkg.CudaLinkedCells()
    tiny = _system(pkg, np.array([[1.0, 1.0, 1.0], [2.0, 1.3, 0.9], [2.0 + 5e-11, 1.3, 0.9]]),
                   (10.0,) * 3, True)
    with pytest.raises(pkg.MinimumSeparationError):
        c.triplet_pass(tiny, ff)
    pos = random_positions(rng, 400, (8.0,) * 3, True)
    for shift in (3e-11, 7e-11):
        p = np.vstack([pos, pos[137] + np.array([0.0, shift, 0.0])])
        s = _system(pkg, p, (8.0,) * 3, True)
        with pytest.raises(pkg.MinimumSeparationError):
            c.triplet_pass(s, ff)


def test_deterministic_passes(pkg):
    s = pkg.systems.CONFIGS["cfg2"].system()
    ff = pkg.ForceField(nu=0.073, cutoff=2.5)
    c = pkg.CudaLinkedCells()
    c.triplet_pass(s, ff)
    a = s.forces_3b.copy()
    e = c.triplet_energy
    c.triplet_pass(s, ff)
    assert np.array_equal(a, s.forces_3b) and e == c.triplet_energy
    c.pair_pass(s, ff)
    b = s.forces_2b.copy()
    c.pair_pass(s, ff)
    assert np.array_equal(b, s.forces_2b)


# --------------------------------------------------------------------------
# BASELINE configs at step 0 (reference scalars / counts / force subsets)
# --------------------------------------------------------------------------
LARGE = ["large_cfg1.npz", "large_cfg2.npz", "large_cfg3_rc2.0.npz", "large_cfg3_rc2.5.npz",
         "large_cfg3_rc3.0.npz", "large_cfg4.npz", "large_cfg5.npz"]


@pytest.mark.parametrize("name", LARGE)
def test_baseline_configs_step0(pkg, name):
    import hashlib

    g = load_golden(name)
    cfg = name.split("_")[1].split(".npz")[0]
    s = pkg.systems.CONFIGS[cfg].system()
    assert hashlib.sha256(s.positions.tobytes()).hexdigest() == str(g["sha"])
    rc3 = float(g["rc3"])
    ff = pkg.ForceField(nu=float(g["nu"]), cutoff=float(g["rc2"]),
                        cutoff_3b=None if rc3 == float(g["rc2"]) else rc3)
    c = pkg.CudaLinkedCells()
    c.pair_pass(s, ff)
    c.triplet_pass(s, ff)
    assert _rel(c.pair_energy, float(g["e2"])) <= ENERGY_TOL
    assert _rel(c.pair_virial, float(g["w2"])) <= VIRIAL_TOL
    assert _rel(c.triplet_energy, float(g["e3"])) <= ENERGY_TOL
    assert _rel(c.triplet_virial, float(g["w3"])) <= VIRIAL_TOL
    if int(g["visits"]) >= 0:
        assert c.triplet_visits == int(g["visits"])
    sub = g["subset"]
    assert np.max(np.abs(s.forces_2b[sub] - g["f2"])) <= FORCE_TOL * float(g["f2_absmax"])
    assert np.max(np.abs(s.forces_3b[sub] - g["f3"])) <= FORCE_TOL * float(g["f3_absmax"])


# --------------------------------------------------------------------------
# device-resident r-RESPA
# --------------------------------------------------------------------------
def _respa_from_golden(pkg, name, container_rc3=None):
    g = load_golden(name)
    s = _system(pkg, g["x0"], g["box"], True, g["v0"])
    rc3 = float(g["cutoff_3b"]) if "cutoff_3b" in g else None
    ff = pkg.ForceField(nu=float(g["nu"]), cutoff=float(g["cutoff"]), cutoff_3b=rc3)
    trace = pkg.respa_run(s, ff, pkg.CudaLinkedCells(),
                          pkg.RespaSchedule(float(g["dt"]), int(g["s"]), int(g["steps"])))
    return g, s, trace


@pytest.mark.parametrize("name", ["respa_cfg1.npz", "respa_small_s3.npz", "respa_split_rc3.npz"])
def test_respa_trajectory_matches_reference(pkg, name):
    g, s, trace = _respa_from_golden(pkg, name)
    assert np.max(np.abs(s.positions - g["x"])) <= 1e-10
    assert np.max(np.abs(s.velocities - g["v"])) <= 1e-10
    assert list(trace.iterations) == [int(v) for v in g["t_iterations"]]
    for got, ref in ((trace.total, g["t_total"]), (trace.potential_3b, g["t_p3"]),
                     (trace.kinetic, g["t_kinetic"])):
        assert max(_rel(a, b) for a, b in zip(got, ref)) <= 1e-10


def test_respa_cfg2_matches_reference(pkg):
    g = load_golden("respa_cfg2.npz")
    s = pkg.systems.CONFIGS["cfg2"].system()
    ff = pkg.ForceField(nu=float(g["nu"]), cutoff=float(g["cutoff"]))
    trace = pkg.respa_run(s, ff, pkg.CudaLinkedCells(), pkg.RespaSchedule(0.001, 5, 100))
    sub = g["subset"]
    assert np.max(np.abs(s.positions[sub] - g["x"])) <= 1e-10
    assert np.max(np.abs(s.velocities[sub] - g["v"])) <= 1e-10
    assert max(_rel(a, b) for a, b in zip(trace.total, g["t_total"])) <= 1e-10
    assert np.all(s.positions >= 0.0) and np.all(s.positions < s.box)


def test_respa_graph_and_eager_identical(pkg):
    base = pkg.systems.fcc_system(6, temperature=0.9, seed=5, vseed=6)
    ff = pkg.ForceField(nu=0.073, cutoff=2.5)
    a, b = base.copy(), base.copy()
    ta = pkg.respa_run(a, ff, pkg.CudaLinkedCells(), pkg.RespaSchedule(0.001, 5, 40), use_graph=True)
    tb = pkg.respa_run(b, ff, pkg.CudaLinkedCells(), pkg.RespaSchedule(0.001, 5, 40), use_graph=False)
    assert np.array_equal(a.positions, b.positions) and np.array_equal(a.velocities, b.velocities)
    assert ta.total == tb.total


def test_verlet_skin_rows_match_rebuild_every_step(pkg):
    """Rows built at rc + skin and rebuilt on the displacement criterion give
    the trajectory of a rebuild-every-step run (only summation order moves)."""
    base = pkg.systems.fcc_system(7, temperature=1.5, seed=9, vseed=10)
    ff = pkg.ForceField(nu=0.073, cutoff=2.5)
    a, b = base.copy(), base.copy()
    ta = pkg.respa_run(a, ff, pkg.CudaLinkedCells(), pkg.RespaSchedule(0.002, 5, 300), skin=0.3)
    tb = pkg.respa_run(b, ff, pkg.CudaLinkedCells(), pkg.RespaSchedule(0.002, 5, 300), skin=0.0)
    assert np.max(np.abs(a.positions - b.positions)) <= 1e-10
    assert np.max(np.abs(a.velocities - b.velocities)) <= 1e-10
    assert max(_rel(x, y) for x, y in zip(ta.total, tb.total)) <= 1e-10


def test_row_capacity_overflow_is_detected_and_retried(pkg):
    """A deliberately small row capacity overflows on the device; the run is
    repeated with larger rows and gives the normal trajectory."""
    base = pkg.systems.fcc_system(6, temperature=0.9, seed=12, vseed=13)
    ff = pkg.ForceField(nu=0.073, cutoff=2.5)
    a, b = base.copy(), base.copy()
    ta = pkg.respa_run(a, ff, pkg.CudaLinkedCells(), pkg.RespaSchedule(0.001, 5, 20), capacity=32)
    tb = pkg.respa_run(b, ff, pkg.CudaLinkedCells(), pkg.RespaSchedule(0.001, 5, 20))
    assert np.max(np.abs(a.positions - b.positions)) <= 1e-12
    assert max(_rel(x, y) for x, y in zip(ta.total, tb.total)) <= 1e-12


def test_s1_is_verlet_and_zero_nu_independent_of_s(pkg):
    base = pkg.systems.fcc_system(5, temperature=1.0, seed=2, vseed=3)
    ff = pkg.ForceField(nu=0.4, cutoff=2.5)
    a, b = base.copy(), base.copy()
    pkg.respa_run(a, ff, pkg.CudaLinkedCells(), pkg.RespaSchedule(0.001, 1, 60))
    pkg.verlet_run(b, ff, pkg.CudaLinkedCells(), 0.001, 60)
    assert np.array_equal(a.positions, b.positions) and np.array_equal(a.velocities, b.velocities)
    ff0 = pkg.ForceField(nu=0.0, cutoff=2.5)
    ref = base.copy()
    pkg.verlet_run(ref, ff0, pkg.CudaLinkedCells(), 0.001, 24)
    for s in (2, 4, 12):
        t = base.copy()
        pkg.respa_run(t, ff0, pkg.CudaLinkedCells(), pkg.RespaSchedule(0.001, s, 24))
        assert np.array_equal(t.positions, ref.positions)
        assert np.array_equal(t.velocities, ref.velocities)


def test_hooks_cadence_momentum_and_wrap(pkg, rng):
    pos = random_positions(rng, 60, (6.5,) * 3, True)
    s = _system(pkg, pos, (6.5,) * 3, True)
    pkg.init_velocities(s, 1.2, seed=3)
    seen, mom = [], []

    def hook(it, view, c):
        seen.append(it)
        mom.append(float(np.max(np.abs(view.velocities.sum(axis=0)))))
        with pytest.raises(ValueError):
            view.positions[0, 0] = 1.0

    ff = pkg.ForceField(nu=0.7, cutoff=2.5)
    pkg.respa_run(s, ff, pkg.CudaLinkedCells(), pkg.RespaSchedule(0.002, 3, 36), sample_interval=6,
                  hooks=(hook,))
    assert seen == [0, 6, 12, 18, 24, 30, 36]
    assert max(mom) <= 1e-9
    assert np.all(s.positions >= 0.0) and np.all(s.positions < s.box)
    with pytest.raises(pkg.ValidationError):
        pkg.respa_run(s, ff, pkg.CudaLinkedCells(), pkg.RespaSchedule(0.001, 4, 8), sample_interval=2)


def test_blowup_iterations(pkg):
    """test_integrators.py:146-161 semantics with the GPU container."""
    ff = pkg.ForceField(nu=0.7, cutoff=2.5)
    s = _system(pkg, np.array([[1.0, 1.0, 1.0], [1.0 + 5e-11, 1.0, 1.0]]), (10.0,) * 3, False)
    with pytest.raises(pkg.IntegrationBlowUp) as err:
        pkg.respa_run(s, ff, pkg.CudaLinkedCells(), pkg.RespaSchedule(0.001, 1, 10))
    assert err.value.iteration == 0
    s = _system(pkg, np.array([[1.0, 1.0, 1.0], [40.0, 40.0, 40.0]]), (50.0,) * 3, False)
    s.velocities[0, 0] = 1e307
    with np.errstate(over="ignore"), pytest.raises(pkg.IntegrationBlowUp) as err:
        pkg.respa_run(s, ff, pkg.CudaLinkedCells(), pkg.RespaSchedule(100.0, 1, 10))
    assert err.value.iteration == 1


def test_respa_rejects_host_containers(pkg):
    s = pkg.systems.fcc_system(4)
    with pytest.raises(TypeError):
        pkg.respa_run(s, pkg.ForceField(), object(), pkg.RespaSchedule(0.001, 1, 1))


def test_container_drives_oracle_respa_loop(pkg, oracle):
    """The GPU container is a drop-in for the reference loop: the oracle's
    restatement of respa_run driven by CudaLinkedCells matches the same loop
    driven by the oracle container."""
    base = pkg.systems.fcc_system(5, temperature=0.9, seed=7, vseed=8)
    ff = pkg.ForceField(nu=0.073, cutoff=2.5)
    a = oracle.OracleSystem.from_positions(base.positions, base.box, True, base.velocities)
    b = a.copy()
    ta = oracle.respa_run(a, ff, pkg.CudaLinkedCells(), 0.001, 2, 20)
    tb = oracle.respa_run(b, ff, oracle.OracleLinkedCells(), 0.001, 2, 20)
    assert np.max(np.abs(a.positions - b.positions)) <= 1e-10
    assert max(_rel(x, y) for x, y in zip(ta.total, tb.total)) <= 1e-10


def _domain_system(pkg, kind):
    if kind == "slab":  # liquid block in the middle half of z, vapour outside
        return pkg.systems.slab_system(n_total=2_400, nc=6, seed=3, temperature=0.8, vseed=4)
    return pkg.systems.fcc_system(8, jitter=0.05, seed=21, temperature=1.2, vseed=22)


def _domain_gpu_worker(rank, world, port, dims, out_dir, kind="fcc", halo="peer", tag=""):
    import os as _os

    import torch.distributed as dist

    _os.environ["MASTER_ADDR"] = "127.0.0.1"
    _os.environ["MASTER_PORT"] = str(port)
    if tag == "win":  # the speculative-window protocol over gloo (CUDA tensors)
        _os.environ["RB_DOMAIN_WINDOW_ANY"] = "1"
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2507_11172_b200 as pkg
        from paper_2507_11172_b200.domain_run import domain_respa_run, gpu_backend_factory

        sysm = _domain_system(pkg, kind)
        ff = pkg.ForceField(nu=0.3, cutoff=2.5)
        trace = domain_respa_run(dist, sysm, ff, pkg.RespaSchedule(0.002, 5, 20),
                                 gpu_backend_factory(ff, halo=halo), skin=0.1, dims=dims,
                                 balance=kind == "slab")
        if rank == 0:
            from paper_2507_11172_b200 import domain_run

            np.savez(_os.path.join(out_dir, f"out_{halo}{tag}.npz"), x=sysm.positions,
                     v=sysm.velocities, total=np.array(trace.total),
                     resumes=domain_run.WINDOW_STATS["resumes"],
                     runs=domain_run.WINDOW_STATS["runs"])
    finally:
        dist.destroy_process_group()


def _run_domain_gpu(tmp_path, world, dims, kind, halo, tag=""):
    import socket

    import torch.multiprocessing as mp

    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    mp.start_processes(_domain_gpu_worker,
                       args=(world, port, dims, str(tmp_path), kind, halo, tag),
                       nprocs=world, join=True, start_method="spawn")
    return np.load(tmp_path / f"out_{halo}{tag}.npz")


@pytest.mark.parametrize("world,dims,kind", [(2, (2, 1, 1), "fcc"), (4, (2, 1, 2), "fcc"),
                                             (4, None, "slab")])
def test_domain_decomposed_gpu_kernels_match_single_domain(pkg, tmp_path, world, dims, kind):
    """The windowed-grid kernels (block + halo binning, windowed neighbour
    cells, owned-weighted energies) on the GPU, ranks as host processes
    sharing cuda:0 (votes over gloo, ghosts pulled from the owners' published
    positions through CUDA IPC; no kernel waits on another rank): trajectory
    equals the single-domain device run.  The slab runs with cost-aware
    (uneven) blocks."""
    out = _run_domain_gpu(tmp_path, world, dims, kind, "peer")
    ref = _domain_system(pkg, kind)
    ff = pkg.ForceField(nu=0.3, cutoff=2.5)
    tr = pkg.respa_run(ref, ff, pkg.CudaLinkedCells(), pkg.RespaSchedule(0.002, 5, 20))
    assert np.max(np.abs(out["x"] - ref.positions)) <= 1e-10
    assert np.max(np.abs(out["v"] - ref.velocities)) <= 1e-10
    assert max(_rel(a, b) for a, b in zip(out["total"], tr.total)) <= 1e-10


def test_domain_peer_halo_equals_message_halo(pkg, tmp_path):
    """The peer-memory ghost refresh (rb_respa_drift_publish + rb_halo_pull)
    and pack / point-to-point / unpack move the same bits."""
    a = _run_domain_gpu(tmp_path, 4, (2, 2, 1), "fcc", "peer")
    b = _run_domain_gpu(tmp_path, 4, (2, 2, 1), "fcc", "nccl")
    assert np.array_equal(a["x"], b["x"]) and np.array_equal(a["v"], b["v"])
    assert np.array_equal(a["total"], b["total"])


def test_kick_folded_into_drift_is_bit_identical(pkg, monkeypatch):
    """rb_respa_kick_drift (a step's kick folded into the next drift inside a
    sampling period) gives exactly the separate kick / drift launches."""
    base = pkg.systems.fcc_system(6, temperature=0.9, seed=15, vseed=16)
    ff = pkg.ForceField(nu=0.073, cutoff=2.5)
    out = []
    for fuse in ("1", "0"):
        monkeypatch.setenv("RB_FUSE_KICK", fuse)
        s = base.copy()
        tr = pkg.respa_run(s, ff, pkg.CudaLinkedCells(), pkg.RespaSchedule(0.002, 3, 60),
                           sample_interval=6)
        out.append((s, tr))
    (a, ta), (b, tb) = out
    assert np.array_equal(a.positions, b.positions) and np.array_equal(a.velocities, b.velocities)
    assert np.array_equal(a.forces_2b, b.forces_2b) and ta.total == tb.total


def test_pair_pass_beside_triplet_kernels_is_bit_identical(pkg, monkeypatch):
    """Three-body steps with the pair pass on a parallel graph branch
    (rb_atm_pass_part 1 | LJ, then part 2) give exactly the sequential
    LJ -> rb_atm_pass order: trajectory, forces and the sampled trace."""
    base = pkg.systems.fcc_system(8, temperature=0.9, seed=21, vseed=22)
    ff = pkg.ForceField(nu=0.073, cutoff=2.5)
    out = []
    for overlap in ("1", "0"):
        monkeypatch.setenv("RB_OVERLAP_PAIR", overlap)
        s = base.copy()
        tr = pkg.respa_run(s, ff, pkg.CudaLinkedCells(), pkg.RespaSchedule(0.002, 5, 100),
                           sample_interval=5)
        out.append((s, tr))
    (a, ta), (b, tb) = out
    assert np.array_equal(a.positions, b.positions) and np.array_equal(a.velocities, b.velocities)
    assert np.array_equal(a.forces_2b, b.forces_2b) and np.array_equal(a.forces_3b, b.forces_3b)
    assert ta.total == tb.total and ta.potential_3b == tb.potential_3b


def test_atm_pass_parts_equal_whole_pass(pkg):
    """rb_atm_pass_part(1) + rb_atm_pass_part(2) = rb_atm_pass, bit for bit,
    and part 1 alone leaves every caller-visible output untouched."""
    import torch

    from paper_2507_11172_b200 import grid
    from paper_2507_11172_b200.engine import ForceEngine

    s = pkg.systems.CONFIGS["cfg2"].system()
    eng = ForceEngine(s.n)
    geom = grid.geometry(s.box, None, 2.5, True)
    eng.upload_positions(s.positions)
    eng.reset_status(0)
    eng.bin(geom)
    eng.nlist(geom, 2.5, checked=True)
    f_whole = torch.empty((s.n, 3), dtype=torch.float64, device="cuda")
    eng.atm_kernel(geom, 2.5, 0.073, f_whole, 0)
    whole = [t.clone() for t in (f_whole, eng.e3_rank, eng.w3_rank, eng.v_rank)]
    f_parts = torch.full((s.n, 3), 7.0, dtype=torch.float64, device="cuda")
    for t in (eng.e3_rank, eng.w3_rank):
        t.fill_(5.0)
    eng.v_rank.fill_(3)
    eng.atm_kernel(geom, 2.5, 0.073, f_parts, 0, part=1)
    torch.cuda.synchronize()
    assert bool((f_parts == 7.0).all()) and bool((eng.e3_rank == 5.0).all())
    assert bool((eng.w3_rank == 5.0).all()) and bool((eng.v_rank == 3).all())
    eng.atm_kernel(geom, 2.5, 0.073, f_parts, 0, part=2)
    parts = (f_parts, eng.e3_rank, eng.w3_rank, eng.v_rank)
    assert all(torch.equal(a, b) for a, b in zip(whole, parts))


@pytest.mark.parametrize("n", [1, 1000, 32000, 250000])
def test_sample_sums_equal_separate_reductions(pkg, n):
    """rb_sample's five sums (one launch) are bit-identical to rb_reduce_sumsq
    / rb_reduce_sum of the same arrays (250,000 particles: more than four
    elements per thread)."""
    import torch

    from paper_2507_11172_b200.engine import ForceEngine

    eng = ForceEngine(n)
    gen = torch.Generator(device="cuda").manual_seed(n)
    rnd = lambda *shape: torch.randn(*shape, dtype=torch.float64, device="cuda",  # noqa: E731
                                     generator=gen)
    v = rnd(n, 3)
    for name in ("e2_rank", "w2_rank", "e3_rank", "w3_rank"):
        getattr(eng, name)[:n] = rnd(n)
    eng.sample(v)
    got = eng.scalars[:5].clone()
    eng.sum_f64(v.reshape(-1), 0, square=True, n=3 * n)
    for slot, name in enumerate(("e2_rank", "w2_rank", "e3_rank", "w3_rank"), start=1):
        eng.sum_f64(getattr(eng, name), slot)
    assert torch.equal(got, eng.scalars[:5])


_TINY = np.array([[2.0, 2.0, 2.0], [3.2, 2.0, 2.0], [2.6, 3.0392304845413265, 2.0],
                  [2.6, 2.3464101615137756, 3.0], [5.2, 5.1, 4.9]])


@pytest.mark.parametrize("n", [0, 1, 2, 3, 4, 5])
@pytest.mark.parametrize("periodic", [True, False])
def test_tiny_systems_match_oracle(pkg, oracle, n, periodic):
    """Empty (rejected, as the reference does), single-particle, one-pair and
    one-triplet systems (and a particle out of everyone's range) through the
    container passes and the device r-RESPA loop: same forces, scalars,
    triplet counts and trajectory as the oracle."""
    box = (6.5, 6.5, 6.5)
    pos = _TINY[:n].copy()
    rng = np.random.default_rng(40 + n)
    vel = rng.normal(0.0, 0.5, size=(n, 3))
    ff = pkg.ForceField(nu=0.5, cutoff=2.5)
    if n == 0:  # the reference rejects an empty system on construction (model.py:94-97)
        with pytest.raises(pkg.ValidationError):
            _system(pkg, pos, box, periodic, vel)
        return
    s = _system(pkg, pos, box, periodic, vel)
    c = pkg.CudaLinkedCells()
    c.pair_pass(s, ff)
    c.triplet_pass(s, ff)
    os_ = oracle.OracleSystem.from_positions(pos, np.array(box), periodic, vel)
    off = oracle.OracleForceField(nu=0.5, cutoff=2.5)
    oc = oracle.OracleLinkedCells()
    oc.pair_pass(os_, off)
    oc.triplet_pass(os_, off)
    assert s.forces_2b.shape == (n, 3) and s.forces_3b.shape == (n, 3)
    assert normwise(s.forces_2b, os_.forces_2b) <= FORCE_TOL
    assert normwise(s.forces_3b, os_.forces_3b) <= FORCE_TOL
    assert abs(c.pair_energy - oc.pair_energy) <= ENERGY_TOL * max(1.0, abs(oc.pair_energy))
    assert abs(c.triplet_energy - oc.triplet_energy) <= ENERGY_TOL * max(1.0, abs(oc.triplet_energy))
    assert c.triplet_count == {3: 1, 4: 4, 5: 4}.get(n, 0)
    # the device loop
    a = _system(pkg, pos, box, periodic, vel)
    tr = pkg.respa_run(a, ff, pkg.CudaLinkedCells(), pkg.RespaSchedule(0.002, 2, 20))
    b = oracle.OracleSystem.from_positions(pos, np.array(box), periodic, vel)
    rtr = oracle.respa_run(b, off, oracle.OracleLinkedCells(), 0.002, 2, 20)
    assert list(tr.iterations) == list(rtr.iterations)
    assert np.max(np.abs(a.positions - b.positions), initial=0.0) <= 1e-10
    assert np.max(np.abs(a.velocities - b.velocities), initial=0.0) <= 1e-10
    assert max((abs(x - y) for x, y in zip(tr.total, rtr.total)), default=0.0) <= 1e-10


@pytest.mark.parametrize("k", [2, 3])
def test_pairs_on_the_cutoff_match_oracle(pkg, oracle, k):
    """A simple-cubic lattice with spacing rc / k: many slot pairs sit on the
    cutoff (within rounding), so the fp64 estimate of r_jk^2 is undecided and
    the reference arithmetic settles them (the fix-up rounds of atm_rot.cuh,
    in rotation rounds for k = 2 and in both rotation and A x B cross rounds
    for k = 3, S+(i) ~ 60).  Counts bit-exact, forces normwise <= 1e-10."""
    h = 2.5 / k
    nd = 4 * k
    g = np.arange(nd) * h
    pos = np.stack(np.meshgrid(g, g, g, indexing="ij"), axis=-1).reshape(-1, 3) + 0.25
    pos = pos[np.arange(len(pos)) % 7 != 3]  # vacancies: nonzero forces, pairs stay on rc
    box = (nd * h,) * 3
    ff = pkg.ForceField(nu=0.4, cutoff=2.5)
    s = _system(pkg, pos, box, True)
    c = pkg.CudaLinkedCells()
    c.triplet_pass(s, ff)
    os_ = oracle.OracleSystem.from_positions(pos, np.array(box), True)
    off = oracle.OracleForceField(nu=0.4, cutoff=2.5)
    grid = oracle.build_cell_grid(os_, 2.5)
    f3, e3, _ = oracle.c01_triplet_pass(grid, os_, off)
    assert c.triplet_visits == oracle.triplet_visit_count(grid, os_)
    assert normwise(s.forces_3b, f3) <= FORCE_TOL
    assert abs(c.triplet_energy - e3) <= ENERGY_TOL * abs(e3)


def _domain_world1_worker(rank, world, port, out_dir, window):
    import os as _os

    import torch.distributed as dist

    _os.environ["MASTER_ADDR"] = "127.0.0.1"
    _os.environ["MASTER_PORT"] = str(port)
    _os.environ["RB_DOMAIN_WINDOW"] = str(window)
    import torch

    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        import paper_2507_11172_b200 as pkg
        from paper_2507_11172_b200 import domain_run
        from paper_2507_11172_b200.domain_run import domain_respa_run, gpu_backend_factory

        sysm = pkg.systems.fcc_system(8, jitter=0.05, seed=21, temperature=1.2, vseed=22)
        ff = pkg.ForceField(nu=0.3, cutoff=2.5)
        trace = domain_respa_run(dist, sysm, ff, pkg.RespaSchedule(0.002, 5, 60),
                                 gpu_backend_factory(ff), skin=0.1)
        np.savez(_os.path.join(out_dir, f"w1_{window}.npz"), x=sysm.positions,
                 v=sysm.velocities, total=np.array(trace.total),
                 resumes=domain_run.WINDOW_STATS["resumes"], runs=domain_run.WINDOW_STATS["runs"])
    finally:
        dist.destroy_process_group()


def test_domain_speculative_windows_match_per_step_votes(pkg, tmp_path):
    """World 1 over NCCL: the speculative-window loop (device rebuild vote,
    RB_KIND_REBUILD freeze, one host synchronisation per window, resume at
    the frozen step) and the per-step host vote give bit-identical
    trajectories, equal to the single-GPU loop within 1e-10; the small skin
    puts rebuild requests inside windows."""
    import socket

    import torch.multiprocessing as mp

    outs = {}
    for window in (16, 0):
        with socket.socket() as so:
            so.bind(("127.0.0.1", 0))
            port = so.getsockname()[1]
        mp.start_processes(_domain_world1_worker, args=(1, port, str(tmp_path), window),
                           nprocs=1, join=True, start_method="spawn")
        outs[window] = np.load(tmp_path / f"w1_{window}.npz")
    a, b = outs[16], outs[0]
    assert int(a["runs"]) == 1 and int(a["resumes"]) >= 2 and int(b["runs"]) == 0
    assert np.array_equal(a["x"], b["x"]) and np.array_equal(a["v"], b["v"])
    assert np.array_equal(a["total"], b["total"])
    ref = pkg.systems.fcc_system(8, jitter=0.05, seed=21, temperature=1.2, vseed=22)
    ff = pkg.ForceField(nu=0.3, cutoff=2.5)
    tr = pkg.respa_run(ref, ff, pkg.CudaLinkedCells(), pkg.RespaSchedule(0.002, 5, 60))
    assert np.max(np.abs(a["x"] - ref.positions)) <= 1e-10
    assert max(_rel(x, y) for x, y in zip(a["total"], tr.total)) <= 1e-10


def _domain_blowup_worker(rank, world, port, out_dir, window):
    import os as _os

    import torch.distributed as dist

    _os.environ["MASTER_ADDR"] = "127.0.0.1"
    _os.environ["MASTER_PORT"] = str(port)
    _os.environ["RB_DOMAIN_WINDOW"] = str(window)
    import torch

    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        import paper_2507_11172_b200 as pkg
        from paper_2507_11172_b200.domain_run import domain_respa_run, gpu_backend_factory

        sysm = pkg.systems.fcc_system(6, jitter=0.05, seed=21, temperature=1.2, vseed=22)
        sysm.velocities[5, 1] = np.inf  # its first drift leaves the box: non-finite
        ff = pkg.ForceField(nu=0.3, cutoff=2.5)
        try:
            domain_respa_run(dist, sysm, ff, pkg.RespaSchedule(0.002, 5, 40),
                             gpu_backend_factory(ff), skin=0.1)
            got = (-1, "")
        except pkg.IntegrationBlowUp as exc:
            got = (exc.iteration, str(exc))
        with open(_os.path.join(out_dir, f"blow_{window}.txt"), "w") as f:
            f.write(f"{got[0]}\n{got[1]}\n")
    finally:
        dist.destroy_process_group()


def test_domain_speculative_windows_report_device_errors(pkg, tmp_path):
    """A non-finite state inside a window (the same step's skin check also
    asks for a rebuild: the error must win) stops the windowed loop at the
    iteration the per-step loop and the single-GPU loop report."""
    import socket

    import torch.multiprocessing as mp

    got = {}
    for window in (16, 0):
        with socket.socket() as so:
            so.bind(("127.0.0.1", 0))
            port = so.getsockname()[1]
        mp.start_processes(_domain_blowup_worker, args=(1, port, str(tmp_path), window),
                           nprocs=1, join=True, start_method="spawn")
        lines = (tmp_path / f"blow_{window}.txt").read_text().splitlines()
        got[window] = int(lines[0])
    ref = pkg.systems.fcc_system(6, jitter=0.05, seed=21, temperature=1.2, vseed=22)
    ref.velocities[5, 1] = np.inf
    with pytest.raises(pkg.IntegrationBlowUp) as err:
        pkg.respa_run(ref, pkg.ForceField(nu=0.3, cutoff=2.5), pkg.CudaLinkedCells(),
                      pkg.RespaSchedule(0.002, 5, 40))
    assert got[16] == got[0] == err.value.iteration >= 1


@pytest.mark.parametrize("world,dims", [(2, (2, 1, 1)), (4, (2, 1, 2))])
def test_domain_speculative_windows_multi_rank(pkg, tmp_path, world, dims):
    """The window protocol across ranks (device votes reduced over the ranks,
    the freeze, one agreed decision per window, migration and ghost rebuild
    at the frozen step, peer pulls ordered by the vote's collective) with
    ranks sharing cuda:0 over gloo: bit-identical to the per-step votes."""
    a = _run_domain_gpu(tmp_path, world, dims, "fcc", "peer", tag="win")
    b = _run_domain_gpu(tmp_path, world, dims, "fcc", "peer")
    assert int(a["runs"]) == 1 and int(a["resumes"]) >= 1 and int(b["runs"]) == 0
    assert np.array_equal(a["x"], b["x"]) and np.array_equal(a["v"], b["v"])
    assert np.array_equal(a["total"], b["total"])
