"""Pin the CPU oracle (oracle/) to the reference's own outputs.

tests/golden/*.npz were produced by running the reference package itself
(tests/golden/make_golden.py).  The oracle restates the reference kernels
operation for operation, so these comparisons are BIT-EXACT; only then is the
oracle trusted as the checker of the GPU path.
"""

import glob
import os

import numpy as np
import pytest

from helpers import GOLDEN, load_golden

SMALL = sorted(os.path.basename(p) for p in glob.glob(os.path.join(GOLDEN, "small_*.npz")))


def test_potential_kernels_bit_exact(oracle):
    g = load_golden("potentials.npz")
    lj = np.array([oracle.lj_kernel(r2, 1.0, 1.0) for r2 in g["r2"]])
    assert np.array_equal(lj, g["lj"])
    atm = np.array([oracle.atm_kernel(a, b, c, float(g["nu"])) for a, b, c in g["abc"]])
    assert np.array_equal(atm, g["atm"])


def _system(oracle, g):
    return oracle.OracleSystem.from_positions(g["positions"], g["box"], bool(g["periodic"]))


@pytest.mark.parametrize("name", SMALL)
def test_grid_and_stencils_bit_exact(oracle, name):
    g = load_golden(name)
    sysm = _system(oracle, g)
    grid = oracle.build_cell_grid(sysm, float(g["cutoff"]))
    assert np.array_equal(grid.cells_per_dim, g["cells"])
    assert np.array_equal(grid.cell_size, g["cell_size"])
    assert np.array_equal(grid.cell_start, g["cell_start"])
    assert np.array_equal(grid.cell_particles, g["cell_particles"])
    assert np.array_equal(grid.pair_cells, g["pair_cells"])
    assert np.array_equal(grid.triplet_patterns, g["triplet_patterns"])
    assert np.array_equal(grid.triplet_same_cell, g["triplet_same_cell"])


@pytest.mark.parametrize("name", SMALL)
def test_c01_passes_bit_exact(oracle, name):
    g = load_golden(name)
    sysm = _system(oracle, g)
    ff = oracle.OracleForceField(nu=float(g["nu"]), cutoff=float(g["cutoff"]))
    grid = oracle.build_cell_grid(sysm, ff.cutoff)
    f2, e2, w2 = oracle.c01_pair_pass(grid, sysm, ff)
    assert np.array_equal(f2, g["f2"]) and e2 == float(g["e2"]) and w2 == float(g["w2"])
    f3, e3, w3 = oracle.c01_triplet_pass(grid, sysm, ff)
    assert np.array_equal(f3, g["f3"]) and e3 == float(g["e3"]) and w3 == float(g["w3"])
    assert oracle.triplet_visit_count(grid, sysm) == int(g["visits"])


@pytest.mark.parametrize("name", SMALL)
def test_brute_force_bit_exact(oracle, name):
    g = load_golden(name)
    sysm = _system(oracle, g)
    ff = oracle.OracleForceField(nu=float(g["nu"]), cutoff=float(g["cutoff"]))
    bf2, be2, bw2 = oracle.brute_force_pairs(sysm, ff, cutoff=ff.cutoff)
    assert np.array_equal(bf2, g["bf2"]) and be2 == float(g["be2"]) and bw2 == float(g["bw2"])
    bf3, be3, bw3, count = oracle.brute_force_triplets(sysm, ff, cutoff=ff.cutoff)
    assert np.array_equal(bf3, g["bf3"]) and be3 == float(g["be3"]) and bw3 == float(g["bw3"])
    assert count == int(g["brute_count"]) == int(g["visits"]) // 3


def test_slab_generator_pinned():
    """cfg5 (liquid slab + vapour) is pinned by sha256; its
    scalars are checked on the GPU (test_baseline_configs_step0)."""
    import hashlib

    from paper_2507_11172_b200 import systems

    g = load_golden("large_cfg5.npz")
    s = systems.CONFIGS["cfg5"].system()
    assert s.n == 500_000
    assert hashlib.sha256(s.positions.tobytes()).hexdigest() == str(g["sha"])


def test_generator_and_large_scalars(oracle):
    """cfg1 and cfg2 at step 0: the generator is pinned by sha256 and the
    oracle's scalars / visit counts / force subsets equal the reference's."""
    import hashlib

    from paper_2507_11172_b200 import systems

    for name, cfg in (("large_cfg1.npz", "cfg1"), ("large_cfg2.npz", "cfg2")):
        g = load_golden(name)
        s = systems.CONFIGS[cfg].system()
        assert hashlib.sha256(s.positions.tobytes()).hexdigest() == str(g["sha"])
        sysm = oracle.OracleSystem.from_positions(s.positions, s.box, True)
        ff = oracle.OracleForceField(nu=float(g["nu"]), cutoff=float(g["rc2"]))
        grid = oracle.build_cell_grid(sysm, ff.cutoff)
        f2, e2, w2 = oracle.c01_pair_pass(grid, sysm, ff)
        f3, e3, w3 = oracle.c01_triplet_pass(grid, sysm, ff)
        assert e2 == float(g["e2"]) and w2 == float(g["w2"])
        assert e3 == float(g["e3"]) and w3 == float(g["w3"])
        sub = g["subset"]
        assert np.array_equal(f2[sub], g["f2"]) and np.array_equal(f3[sub], g["f3"])
        assert oracle.triplet_visit_count(grid, sysm) == int(g["visits"])


def test_respa_cfg1_bit_exact(oracle):
    """respa_run restatement: 10 Verlet steps of BASELINE config 1."""
    g = load_golden("respa_cfg1.npz")
    sysm = oracle.OracleSystem.from_positions(g["x0"], g["box"], True, velocities=g["v0"])
    ff = oracle.OracleForceField(nu=float(g["nu"]), cutoff=float(g["cutoff"]))
    trace = oracle.respa_run(sysm, ff, oracle.OracleLinkedCells(), float(g["dt"]), int(g["s"]),
                             int(g["steps"]))
    assert np.array_equal(sysm.positions, g["x"])
    assert np.array_equal(sysm.velocities, g["v"])
    assert np.array_equal(np.array(trace.total), g["t_total"])


def test_respa_small_s3_bit_exact(oracle):
    g = load_golden("respa_small_s3.npz")
    sysm = oracle.OracleSystem.from_positions(g["x0"], g["box"], True, velocities=g["v0"])
    ff = oracle.OracleForceField(nu=float(g["nu"]), cutoff=float(g["cutoff"]))
    trace = oracle.respa_run(sysm, ff, oracle.OracleLinkedCells(), float(g["dt"]), int(g["s"]),
                             int(g["steps"]))
    assert np.array_equal(sysm.positions, g["x"])
    assert np.array_equal(sysm.velocities, g["v"])
    assert np.array_equal(np.array(trace.iterations), g["t_iterations"])
    assert np.array_equal(np.array(trace.potential_3b), g["t_p3"])


def test_respa_split_cutoff_bit_exact(oracle):
    g = load_golden("respa_split_rc3.npz")
    sysm = oracle.OracleSystem.from_positions(g["x0"], g["box"], True, velocities=g["v0"])
    ff = oracle.OracleForceField(nu=float(g["nu"]), cutoff=float(g["cutoff"]))
    oracle.respa_run(sysm, ff, oracle.OracleLinkedCells(rc3=float(g["cutoff_3b"])), float(g["dt"]),
                     int(g["s"]), int(g["steps"]))
    assert np.array_equal(sysm.positions, g["x"])
    assert np.array_equal(sysm.velocities, g["v"])


def _direct_cases():
    g = load_golden("direct.npz")
    return g, [str(n) for n in g["names"]]


def test_direct_sum_bit_exact(oracle):
    """DirectSum restatement (containers.py:663-739, 852-875) vs the reference."""
    g, names = _direct_cases()
    off = oracle.OracleForceField(nu=float(g["nu"]), cutoff=2.5)
    for name in names:
        s = oracle.OracleSystem.from_positions(g[f"{name}__pos"], g[f"{name}__box"], False)
        f2, e2, w2 = oracle.direct_sum_pairs(s, off)
        f3, e3, w3 = oracle.direct_sum_triplets(s, off)
        assert np.array_equal(f2, g[f"{name}__f2"]) and np.array_equal(f3, g[f"{name}__f3"])
        assert (e2, w2, e3, w3) == (float(g[f"{name}__e2"]), float(g[f"{name}__w2"]),
                                    float(g[f"{name}__e3"]), float(g[f"{name}__w3"]))


def test_direct_sum_rejects_periodic(oracle):
    s = oracle.OracleSystem.from_positions(np.zeros((3, 3)) + [[0, 0, 0], [1, 0, 0], [0, 1, 0]],
                                           (5.0, 5.0, 5.0), True)
    with pytest.raises(oracle.OracleValidationError):
        oracle.direct_sum_pairs(s, oracle.OracleForceField())


def test_distance_histogram_bit_exact(oracle):
    """RDF pair counts (observables.py:143-177) vs the reference."""
    g = load_golden("rdf.npz")
    for name in [str(n) for n in g["names"]]:
        frames = int(g[f"{name}__frames"])
        counts = sum(oracle.distance_histogram(g[f"{name}__frame{i}"], g[f"{name}__box"],
                                               float(g[f"{name}__r_max"]), int(g[f"{name}__bins"]))
                     for i in range(frames))
        assert np.array_equal(counts, g[f"{name}__counts"])
