"""DirectSum on the GPU: rb_direct_pairs / rb_direct_triplets
against the reference's own outputs (tests/golden/direct.npz, made by
respamd.containers.direct_sum_*) and the bit-pinned oracle, plus the
reference's DirectSum tests (test_containers.py:188-257) on the GPU path.

Tolerances as in test_gpu_parity.py: forces normwise 1e-10, energies 1e-10
relative, virials 1e-9 relative.
"""

import itertools

import numpy as np
import pytest

from helpers import TEST_SEED, load_golden, normwise, random_positions

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pkg():
    import paper_2507_11172_b200 as p
    from paper_2507_11172_b200 import _lib

    _lib.require_device()
    return p


def _rel(a, b):
    return abs(a - b) / max(1.0, abs(b))


def _system(pkg, pos, edge, periodic=False):
    s = pkg.ParticleSystem.empty(len(pos), (edge,) * 3, periodic=periodic)
    s.positions[:] = pos
    return s


def test_direct_sum_matches_reference(pkg):
    g = load_golden("direct.npz")
    ff = pkg.ForceField(nu=float(g["nu"]), cutoff=2.5)
    for name in [str(n) for n in g["names"]]:
        s = _system(pkg, g[f"{name}__pos"], float(g[f"{name}__box"][0]))
        f2, e2, w2 = pkg.direct_sum_pairs(s, ff)
        f3, e3, w3 = pkg.direct_sum_triplets(s, ff)
        assert normwise(f2, g[f"{name}__f2"]) <= 1e-10, name
        assert normwise(f3, g[f"{name}__f3"]) <= 1e-10, name
        assert _rel(e2, float(g[f"{name}__e2"])) <= 1e-10
        assert _rel(e3, float(g[f"{name}__e3"])) <= 1e-10
        assert _rel(w2, float(g[f"{name}__w2"])) <= 1e-9
        assert _rel(w3, float(g[f"{name}__w3"])) <= 1e-9


@pytest.mark.parametrize("n", [2, 3, 5, 257, 258, 600])
def test_direct_sum_against_oracle_sizes(pkg, oracle, n):
    """Both enumeration paths of the triplet pass (followers m < 256: one
    round per window; m >= 256: 256-pair windows across rounds)."""
    rng = np.random.default_rng(TEST_SEED + n)
    edge = max(4.0, (n / 0.5) ** (1 / 3))
    pos = random_positions(rng, n, (edge,) * 3, False)
    ff = pkg.ForceField(nu=0.5, cutoff=2.5)
    s = _system(pkg, pos, edge)
    f2, e2, w2 = pkg.direct_sum_pairs(s, ff)
    f3, e3, w3 = pkg.direct_sum_triplets(s, ff)
    os_ = oracle.OracleSystem.from_positions(pos, (edge,) * 3, False)
    off = oracle.OracleForceField(nu=0.5, cutoff=2.5)
    rf2, re2, rw2 = oracle.direct_sum_pairs(os_, off)
    rf3, re3, rw3 = oracle.direct_sum_triplets(os_, off)
    assert normwise(f2, rf2) <= 1e-10 and normwise(f3, rf3) <= 1e-10
    assert _rel(e2, re2) <= 1e-10 and _rel(e3, re3) <= 1e-10
    assert _rel(w2, rw2) <= 1e-9 and _rel(w3, rw3) <= 1e-9


def test_four_particle_interaction_counts(pkg):
    """test_containers.py:189-207: energies equal the sums over the 6 pairs
    and 4 triplets of closed forms."""
    pos = np.array([[0.0, 0.0, 0.0], [1.2, 0.0, 0.0], [0.0, 1.3, 0.0], [0.0, 0.0, 1.4]])
    ff = pkg.ForceField(nu=0.7, cutoff=2.5)
    s = _system(pkg, pos, 50.0)
    _, e2, _ = pkg.direct_sum_pairs(s, ff)
    _, e3, _ = pkg.direct_sum_triplets(s, ff)

    def lj(r):
        return 4.0 * ((1.0 / r) ** 12 - (1.0 / r) ** 6)

    def atm(a, b, c):
        ab, ac, bc = b - a, c - a, c - b
        rab, rac, rbc = np.linalg.norm(ab), np.linalg.norm(ac), np.linalg.norm(bc)
        cos_a = np.dot(ab, ac) / (rab * rac)
        cos_b = np.dot(-ab, bc) / (rab * rbc)
        cos_c = np.dot(-ac, -bc) / (rac * rbc)
        return 0.7 * (1.0 + 3.0 * cos_a * cos_b * cos_c) / (rab * rac * rbc) ** 3

    ref2 = sum(lj(np.linalg.norm(pos[i] - pos[j])) for i, j in itertools.combinations(range(4), 2))
    ref3 = sum(atm(pos[i], pos[j], pos[k]) for i, j, k in itertools.combinations(range(4), 3))
    assert e2 == pytest.approx(ref2, rel=1e-12)
    assert e3 == pytest.approx(ref3, rel=1e-12)


def test_two_particle_action_reaction(pkg):
    """test_containers.py:209-213: the net force is exactly zero."""
    s = _system(pkg, np.array([[1.0, 1.0, 1.0], [2.3, 1.8, 1.1]]), 10.0)
    f, _, _ = pkg.direct_sum_pairs(s, pkg.ForceField())
    assert np.max(np.abs(f.sum(axis=0))) == 0.0


def test_linked_cells_with_huge_cutoff_equals_direct_sum(pkg, rng):
    """test_containers.py:235-249 on the two GPU containers."""
    for n in (40, 80, 100):
        pos = random_positions(rng, n, (6.0,) * 3, False)
        s = _system(pkg, pos, 6.0)
        diag = float(np.linalg.norm(s.box))
        ff_all = pkg.ForceField(nu=0.7, cutoff=diag)
        ds, lc = pkg.CudaDirectSum(), pkg.CudaLinkedCells()
        a, b = s.copy(), s.copy()
        ds.pair_pass(a, ff_all)
        ds.triplet_pass(a, ff_all)
        lc.pair_pass(b, ff_all)
        lc.triplet_pass(b, ff_all)
        assert np.max(np.abs(a.forces_2b - b.forces_2b)) <= 1e-9
        assert np.max(np.abs(a.forces_3b - b.forces_3b)) <= 1e-9
        assert ds.pair_energy == pytest.approx(lc.pair_energy, rel=1e-9)
        assert ds.triplet_energy == pytest.approx(lc.triplet_energy, rel=1e-9)


def test_direct_sum_guard_and_determinism(pkg):
    rng = np.random.default_rng(TEST_SEED)
    pos = random_positions(rng, 300, (9.0,) * 3, False)
    s = _system(pkg, pos, 9.0)
    ff = pkg.ForceField(nu=0.3)
    c = pkg.make_container("direct_sum")
    c.triplet_pass(s, ff)
    first = s.forces_3b.copy()
    c.triplet_pass(s, ff)
    assert np.array_equal(first, s.forces_3b)
    pos2 = pos.copy()
    pos2[7] = pos2[3]  # coincident particles
    s2 = _system(pkg, pos2, 9.0)
    with pytest.raises(pkg.MinimumSeparationError):
        pkg.direct_sum_pairs(s2, ff)
    with pytest.raises(pkg.MinimumSeparationError):
        pkg.direct_sum_triplets(s2, ff)
    c.triplet_pass(s, pkg.ForceField(nu=0.0))
    assert not s.forces_3b.any() and c.triplet_energy == 0.0


def test_respa_with_direct_sum_matches_oracle(pkg, oracle):
    """The device r-RESPA loop driving DirectSum (graph replay and eager)
    against the oracle's respa_run with the DirectSum restatement."""
    rng = np.random.default_rng(TEST_SEED + 5)
    n, edge = 80, 7.0
    pos = random_positions(rng, n, (edge,) * 3, False)
    vel = rng.normal(0.0, 0.5, (n, 3))
    vel -= vel.mean(axis=0)
    ff = pkg.ForceField(nu=0.4)
    sched = pkg.RespaSchedule(0.002, 3, 30)
    runs = []
    for graph in (True, False):
        s = _system(pkg, pos, edge)
        s.velocities[:] = vel
        runs.append((s, pkg.respa_run(s, ff, pkg.CudaDirectSum(), sched, use_graph=graph)))
    os_ = oracle.OracleSystem.from_positions(pos, (edge,) * 3, False, vel)
    otr = oracle.respa_run(os_, oracle.OracleForceField(nu=0.4), oracle.OracleDirectSum(), 0.002,
                           3, 30)
    (sg, tg), (se, te) = runs
    assert np.array_equal(sg.positions, se.positions) and tg.total == te.total
    assert np.max(np.abs(sg.positions - os_.positions)) <= 1e-10
    assert np.max(np.abs(sg.velocities - os_.velocities)) <= 1e-10
    assert list(tg.iterations) == list(otr.iterations)
    assert max(_rel(a, b) for a, b in zip(tg.total, otr.total)) <= 1e-10


def _dist_worker(rank, world, port, out_dir):
    import os as _os

    import torch.distributed as dist

    _os.environ["MASTER_ADDR"] = "127.0.0.1"
    _os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2507_11172_b200 as pkg
        from paper_2507_11172_b200.direct_dist import DistributedDirectSum

        rng = np.random.default_rng(TEST_SEED + 77)
        pos = random_positions(rng, 400, (10.0,) * 3, False)
        s = pkg.ParticleSystem.empty(400, (10.0,) * 3, periodic=False)
        s.positions[:] = pos
        c = DistributedDirectSum(dist)
        ff = pkg.ForceField(nu=0.5)
        c.pair_pass(s, ff)
        c.triplet_pass(s, ff)
        np.savez(_os.path.join(out_dir, f"r{rank}.npz"), f2=s.forces_2b, f3=s.forces_3b,
                 e=np.array([c.pair_energy, c.pair_virial, c.triplet_energy, c.triplet_virial]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_distributed_direct_sum_matches_single(pkg, tmp_path, world):
    """Ranks as processes sharing cuda:0 (gloo exchange): every rank holds the
    same result, equal to the one-GPU pass to rounding."""
    import socket

    import torch.multiprocessing as mp

    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    mp.start_processes(_dist_worker, args=(world, port, str(tmp_path)), nprocs=world, join=True,
                       start_method="spawn")
    outs = [np.load(tmp_path / f"r{r}.npz") for r in range(world)]
    for o in outs[1:]:
        assert np.array_equal(o["f2"], outs[0]["f2"]) and np.array_equal(o["f3"], outs[0]["f3"])
        assert np.array_equal(o["e"], outs[0]["e"])
    rng = np.random.default_rng(TEST_SEED + 77)
    pos = random_positions(rng, 400, (10.0,) * 3, False)
    s = _system(pkg, pos, 10.0)
    ff = pkg.ForceField(nu=0.5)
    f2, e2, w2 = pkg.direct_sum_pairs(s, ff)
    f3, e3, w3 = pkg.direct_sum_triplets(s, ff)
    assert normwise(outs[0]["f2"], f2) <= 1e-13 and normwise(outs[0]["f3"], f3) <= 1e-13
    for got, ref in zip(outs[0]["e"], (e2, w2, e3, w3)):
        assert _rel(got, ref) <= 1e-12
