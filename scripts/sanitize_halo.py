"""compute-sanitizer workload for the fused slab halos (k_diffusion_slab_edges and
k_diffusion_slab_halo2): two ranks share cuda:0 (gloo control plane, CUDA IPC mailboxes),
p2p SlabDiffusion step() and run(), checked against the single-device run. Run as
    compute-sanitizer --tool memcheck --target-processes all python scripts/sanitize_halo.py
"""
from __future__ import annotations

import os
import socket
import sys

import numpy as np
import torch
import torch.multiprocessing as mp

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def worker(rank, world, port, q):
    import torch.distributed as dist

    import paper_2411_18889_b200 as b2
    from paper_2411_18889_b200.distributed import SlabDiffusion

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    shape, args, steps = (8, 20, 64), (0.1, 0.12, 0.09, 1e-3, 1.0), 4
    f0 = torch.from_numpy(np.random.default_rng(3).random(shape, dtype=np.float32))
    nl = shape[0] // world
    sim = SlabDiffusion(f0[rank * nl:(rank + 1) * nl].contiguous().cuda(), *args, transport="p2p")
    sim.step(steps)
    sim.run(4)  # two steps per exchange: b2_diffusion3d_slab_halo2 push / ingest
    torch.cuda.synchronize()
    parts = [None] * world
    dist.all_gather_object(parts, sim.f.cpu().numpy())
    sim.close()
    if rank == 0:
        ref = b2.Diffusion3D(f0.cuda(), *args).run(steps + 4).cpu().numpy()
        q.put(bool(np.array_equal(np.concatenate(parts).view(np.uint32), ref.view(np.uint32))))
    dist.destroy_process_group()


if __name__ == "__main__":
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    mp.spawn(worker, args=(2, port, q), nprocs=2, join=True)
    ok = q.get()
    print("halo ok" if ok else "halo MISMATCH")
    sys.exit(0 if ok else 1)
