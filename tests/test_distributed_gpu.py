"""GPU: the distributed classes on the CUDA kernels through NCCL (world_size 1 on the one
GPU gpurun gives; the multi-rank exchange logic is covered on CPU by test_distributed.py).

Checks that the sharded driver (NCCL in-place all-gather + partials + fused update) and
the slab driver (comm stream, interior/boundary split) reproduce the single-device
paths bit for bit.
"""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, port, out):
    import torch.distributed as dist

    import paper_2411_18889_b200 as b2
    from paper_2411_18889_b200.distributed import ShardedLeapfrog, SlabDiffusion

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    n, eps, dt = 8192, 2.0 ** -6, 2.0 ** -7
    pos, vel = b2.plummer(n, 42)
    sh = ShardedLeapfrog(pos, vel, eps, dt)
    sh.step(4)
    lf = b2.Leapfrog(pos.clone(), vel.clone(), eps, dt)
    lf.step(4)
    f = b2.init_grid(16, 24, 32, seed=2)
    sd = SlabDiffusion(f, 0.1, 0.1, 0.1, 1e-3, 1.0)
    sd.step(3)
    ref = b2.Diffusion3D(f.clone(), 0.1, 0.1, 0.1, 1e-3, 1.0)
    ref.run(3)
    torch.cuda.synchronize()
    np.savez(out, sp=sh.pos.cpu().numpy(), sv=sh.vel.cpu().numpy(), sa=sh.acc.cpu().numpy(),
             lp=lf.pos.cpu().numpy(), lv=lf.vel.cpu().numpy(), la=lf.acc.cpu().numpy(),
             sd=sd.f.cpu().numpy(), rd=ref.field.cpu().numpy())
    dist.destroy_process_group()


def test_distributed_drivers_match_single_device(tmp_path):
    import torch.multiprocessing as mp

    out = tmp_path / "o.npz"
    mp.spawn(_worker, args=(_port(), str(out)), nprocs=1, join=True)
    z = np.load(out)
    for a, b in (("sp", "lp"), ("sv", "lv"), ("sa", "la"), ("sd", "rd")):
        assert np.array_equal(z[a].view(np.uint32), z[b].view(np.uint32)), a
