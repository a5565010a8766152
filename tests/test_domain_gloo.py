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


def _system():
    from paper_2507_11172_b200 import systems

    return systems.fcc_system(8, jitter=0.05, seed=21, temperature=1.2, vseed=22)


def _worker(rank, world, port, dims, steps, s, out_dir, skin):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from domain_backend import NumpyBackend

        from paper_2507_11172_b200 import ForceField, RespaSchedule
        from paper_2507_11172_b200.domain_run import domain_respa_run

        sysm = _system()
        ff = ForceField(nu=0.3, cutoff=2.5)
        trace = domain_respa_run(dist, sysm, ff, RespaSchedule(0.002, s, steps),
                                 lambda dec, n, rb: NumpyBackend(ff, sysm.box), skin=skin,
                                 dims=dims)
        if rank == 0:
            np.savez(os.path.join(out_dir, "out.npz"), x=sysm.positions, v=sysm.velocities,
                     f2=sysm.forces_2b, f3=sysm.forces_3b, total=np.array(trace.total),
                     it=np.array(trace.iterations))
    finally:
        dist.destroy_process_group()


def _oracle_run(steps, s):
    from oracle import oracle as o

    sysm = _system()
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
