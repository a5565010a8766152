"""Domain decomposition on CPU with gloo (world sizes 2 and 4).

The exchange logic (migration, staged ghosts, per-step refresh, rank-order
sums) of paper_2507_11172_b200/domain.py runs with a numpy force backend;
the decomposed r-RESPA trajectory must equal the single-domain oracle's
(oracle/ C01 restatement, bit-pinned to the reference) within 1e-10.
"""

import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, HERE)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _system(kind="fcc"):
    from paper_2507_11172_b200 import systems

    if kind == "slab":  # liquid block in the middle half of z, vapour outside
        return systems.slab_system(n_total=560, nc=4, seed=3, temperature=0.8, vseed=4)
    return systems.fcc_system(8, jitter=0.05, seed=21, temperature=1.2, vseed=22)


def _worker(rank, world, port, dims, steps, s, out_dir, skin, kind="fcc", balance=False):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from domain_backend import NumpyBackend

        from paper_2507_11172_b200 import ForceField, RespaSchedule
        from paper_2507_11172_b200.domain_run import domain_respa_run

        sysm = _system(kind)
        ff = ForceField(nu=0.3, cutoff=2.5)
        seen = {}

        def factory(dec, n, rb):
            seen["dims"], seen["bounds"] = dec.dims, dec.bounds
            return NumpyBackend(ff, sysm.box)

        trace = domain_respa_run(dist, sysm, ff, RespaSchedule(0.002, s, steps), factory,
                                 skin=skin, dims=dims, balance=balance)
        if rank == 0:
            np.savez(os.path.join(out_dir, "out.npz"), x=sysm.positions, v=sysm.velocities,
                     f2=sysm.forces_2b, f3=sysm.forces_3b, total=np.array(trace.total),
                     it=np.array(trace.iterations), dims=np.array(seen["dims"]),
                     zbounds=np.array(seen["bounds"][2]))
    finally:
        dist.destroy_process_group()


def _oracle_run(steps, s, kind="fcc"):
    from oracle import oracle as o

    sysm = _system(kind)
    osys = o.OracleSystem.from_positions(sysm.positions, sysm.box, True, sysm.velocities)
    off = o.OracleForceField(nu=0.3, cutoff=2.5)
    trace = o.respa_run(osys, off, o.OracleLinkedCells(), 0.002, s, steps)
    return osys, trace


@pytest.mark.parametrize("world,dims,skin", [(2, (2, 1, 1), 0.3), (4, (2, 2, 1), 0.3),
                                             (2, (1, 1, 2), 0.0)])
def test_decomposed_respa_matches_single_domain(tmp_path, world, dims, skin):
    """skin 0 rebuilds (migration + ghosts) every step; 0.3 refreshes ghosts."""
    steps, s = 10, 5
    port = _free_port()
    mp.start_processes(_worker, args=(world, port, dims, steps, s, str(tmp_path), skin),
                       nprocs=world, join=True, start_method="spawn")
    out = np.load(tmp_path / "out.npz")
    ref, rtrace = _oracle_run(steps, s)
    assert np.max(np.abs(out["x"] - ref.positions)) <= 1e-10
    assert np.max(np.abs(out["v"] - ref.velocities)) <= 1e-10
    assert np.max(np.abs(out["f3"] - ref.forces_3b)) <= 1e-10
    assert list(out["it"]) == list(rtrace.iterations)
    rel = np.abs(out["total"] - np.array(rtrace.total)) / np.abs(np.array(rtrace.total))
    assert np.max(rel) <= 1e-10


def test_balanced_slab_matches_single_domain(tmp_path):
    """Cost-aware blocks (domain.balanced_layout) on a liquid slab: the z cuts
    crowd into the liquid, and the trajectory still equals the oracle's."""
    world, steps, s = 4, 10, 5
    port = _free_port()
    mp.start_processes(_worker, args=(world, port, None, steps, s, str(tmp_path), 0.3, "slab",
                                      True), nprocs=world, join=True, start_method="spawn")
    out = np.load(tmp_path / "out.npz")
    assert tuple(out["dims"]) == (1, 1, 4)
    widths = np.diff(out["zbounds"])
    assert widths.max() > widths.min()  # uneven: thin blocks in the liquid
    ref, rtrace = _oracle_run(steps, s, "slab")
    assert np.max(np.abs(out["x"] - ref.positions)) <= 1e-10
    assert np.max(np.abs(out["v"] - ref.velocities)) <= 1e-10
    assert list(out["it"]) == list(rtrace.iterations)
    rel = np.abs(out["total"] - np.array(rtrace.total)) / np.abs(np.array(rtrace.total))
    assert np.max(rel) <= 1e-10


def test_balanced_bounds_is_optimal():
    """Exact minimax cut against brute force, with the width limits."""
    import itertools

    from paper_2507_11172_b200.domain import balanced_bounds

    rng = np.random.default_rng(5)
    for trial in range(40):
        n = int(rng.integers(4, 11))
        parts = int(rng.integers(1, 4))
        prof = rng.integers(0, 6, size=n).astype(np.float64)
        best = None
        for cuts in itertools.combinations(range(1, n), parts - 1):
            b = (0,) + cuts + (n,)
            w = np.diff(b)
            if parts > 1 and (w.min() < 1 or w.max() > n - 2):
                continue
            v = max(prof[b[k]:b[k + 1]].sum() for k in range(parts))
            best = v if best is None else min(best, v)
        if best is None:
            with pytest.raises(ValueError):
                balanced_bounds(prof, parts)
            continue
        b = balanced_bounds(prof, parts)
        w = np.diff(b)
        assert b[0] == 0 and b[-1] == n and w.min() >= 1
        assert parts == 1 or w.max() <= n - 2
        assert max(prof[b[k]:b[k + 1]].sum() for k in range(parts)) == best


def test_balanced_layout_evens_the_slab_load():
    from paper_2507_11172_b200 import systems
    from paper_2507_11172_b200.domain import (Decomposition, auto_dims, balanced_layout,
                                              block_costs, cell_costs, cell_occupancy)
    from paper_2507_11172_b200.grid import geometry

    sysm = systems.slab_system(n_total=14_000, nc=12, seed=2)
    geom = geometry(sysm.box, None, 2.8, True)
    occ = cell_occupancy(sysm.positions, geom)
    costs = cell_costs(sysm.positions, geom, 0.29 / 5)
    assert occ.sum() == sysm.positions.shape[0]
    even = Decomposition(sysm.box, 2.8, 8, 0, auto_dims(8, geom.cells))
    dims, bounds = balanced_layout(costs, 8, occ)
    before = block_costs(costs, even.dims, even.bounds, occ)
    after = block_costs(costs, dims, bounds, occ)
    # 7 x 7 x 29 cells: whole-layer cuts limit the balance
    assert before.max() / before.mean() > 2.0
    assert after.max() < 0.6 * before.max() and after.max() / after.mean() < 1.3
    # the layout is usable: every particle gets exactly one owner
    owners = np.concatenate([np.nonzero(Decomposition(sysm.box, 2.8, 8, r, dims, bounds)
                                        .owner_rank(sysm.positions) == r)[0] for r in range(8)])
    assert np.array_equal(np.sort(owners), np.arange(sysm.positions.shape[0]))
    with pytest.raises(ValueError):
        Decomposition(sysm.box, 2.8, 2, 0, (1, 1, 2), [[0, geom.cells[0]], [0, geom.cells[1]],
                                                       [0, 0, geom.cells[2]]])


def test_decomposition_geometry():
    from paper_2507_11172_b200.domain import Decomposition, auto_dims
    from paper_2507_11172_b200 import systems

    box = np.full(3, 80 * systems.FCC_A)
    assert auto_dims(8, (48, 48, 48)) == (2, 2, 2)
    assert auto_dims(2, (48, 48, 48)) in ((2, 1, 1), (1, 2, 1), (1, 1, 2))
    dec = Decomposition(box, 2.8, 8, 5)
    assert dec.dims == (2, 2, 2) and dec.coord == (1, 0, 1)
    w = dec.window()
    assert w.cells == (dec.hi[0] - dec.lo[0] + 2,) * 3
    # every particle has exactly one owner
    rng = np.random.default_rng(0)
    pos = rng.uniform(0, box, size=(5000, 3))
    owners = dec.owner_rank(pos)
    assert owners.min() >= 0 and owners.max() < 8
    offs = w.offsets()
    assert offs.shape == (27, 3) and offs.min() == -1


@pytest.mark.parametrize("world,dims,balanced", [(1, None, False), (2, (2, 1, 1), False),
                                                 (8, (2, 2, 2), False), (4, (1, 1, 4), True)])
def test_device_decomposition_maps_equal_numpy(world, dims, balanced):
    """The rebuild's torch cell / block / owner maps and the window population
    (domain.Decomposition.*_t, run on the payload's device) equal the numpy
    restatement bit for bit, on positions that include the box faces, cell
    boundaries and the wrapped coordinate 0."""
    from paper_2507_11172_b200 import systems
    from paper_2507_11172_b200.domain import Decomposition

    s = systems.fcc_system(16, jitter=0.05, seed=3)  # 9 cells per dimension at 2.8
    pos = s.positions.copy()
    box = np.asarray(s.box, dtype=np.float64)
    dec0 = Decomposition(box, 2.8, world, 0, dims)
    n = np.asarray(dec0.geom.cells)
    edge = np.stack([np.zeros(3), box * (1.0 - 1e-16), box / n, 2 * box / n * (1 - 1e-15)])
    pos = np.concatenate([pos, edge], axis=0)
    bounds = None
    if balanced:  # uneven cuts along z
        nz = int(n[2])
        bounds = [[0, int(n[0])], [0, int(n[1])], [0, 2, 4, 6, nz]]
    t = torch.as_tensor(pos)
    for rank in range(world):
        dec = Decomposition(box, 2.8, world, rank, dims if not balanced else (1, 1, 4), bounds)
        cn = dec.cells_of(pos)
        ct = dec.cells_of_t(t)
        assert np.array_equal(cn, ct.numpy())
        bn = dec.block_of(cn)
        for d in range(3):
            assert np.array_equal(bn[:, d], dec.block_coord_t(ct[:, d], d).numpy())
        assert np.array_equal(dec.owner_rank(pos), dec.owner_rank_t(t).numpy())
        assert dec.window_count(pos) == dec.window_count_t(t)
