"""The decomposed loop over NCCL on distinct GPUs (one process per GPU, as
bench.py --gpus N runs it): skipped unless the box has at least two GPUs.
The trajectory must equal the single-GPU device run."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _port():
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def _worker(rank, world, port, out, halo):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world)
    try:
        import paper_2507_11172_b200 as pkg
        from paper_2507_11172_b200.domain_run import domain_respa_run, gpu_backend_factory

        s = pkg.systems.fcc_system(10, jitter=0.03, seed=31, temperature=1.1, vseed=32)
        ff = pkg.ForceField(nu=0.2, cutoff=2.5)
        tr = domain_respa_run(dist, s, ff, pkg.RespaSchedule(0.002, 5, 40),
                              gpu_backend_factory(ff, halo=halo))
        if rank == 0:
            np.savez(out, x=s.positions, v=s.velocities, total=np.array(tr.total))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,halo", [(2, "peer"), (2, "nccl"), (4, "peer"), (8, "peer")])
def test_nccl_decomposed_run_matches_single_gpu(tmp_path, world, halo):
    import torch
    import torch.multiprocessing as mp

    if torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs (this box has {torch.cuda.device_count()})")
    out = str(tmp_path / "out.npz")
    mp.start_processes(_worker, args=(world, _port(), out, halo), nprocs=world, join=True,
                       start_method="spawn")
    got = np.load(out)
    import paper_2507_11172_b200 as pkg

    ref = pkg.systems.fcc_system(10, jitter=0.03, seed=31, temperature=1.1, vseed=32)
    ff = pkg.ForceField(nu=0.2, cutoff=2.5)
    tr = pkg.respa_run(ref, ff, pkg.CudaLinkedCells(), pkg.RespaSchedule(0.002, 5, 40))
    assert np.max(np.abs(got["x"] - ref.positions)) <= 1e-10
    assert np.max(np.abs(got["v"] - ref.velocities)) <= 1e-10
    assert max(abs(a - b) / max(1.0, abs(b)) for a, b in zip(got["total"], tr.total)) <= 1e-10
