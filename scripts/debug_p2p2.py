import os, sys, socket
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch, torch.multiprocessing as mp

def worker(rank, world, port, mode, out):
    import torch.distributed as dist
    import paper_2411_18889_b200 as b2
    from paper_2411_18889_b200.distributed import ShardedLeapfrog
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n = 8192
    pos, vel = b2.plummer_numpy(n, 8)
    nl = n // world
    sim = ShardedLeapfrog(torch.from_numpy(pos[rank*nl:(rank+1)*nl]).cuda(), torch.from_numpy(vel[rank*nl:(rank+1)*nl]).cuda(), 2.0**-6, 2.0**-7, transport="p2p")
    init_acc = sim.acc.cpu().numpy(); init_all = sim.pos_all.cpu().numpy()
    for s in range(3):
        if mode == "sync":
            torch.cuda.synchronize(); dist.barrier()
        sim.step(1, close=(s == 2))
    torch.cuda.synchronize(); dist.barrier()
    parts = [None] * world
    dist.all_gather_object(parts, (sim.pos.cpu().numpy(), init_acc, init_all))
    sim.close()
    if rank == 0:
        lf = b2.Leapfrog(torch.from_numpy(pos).cuda(), torch.from_numpy(vel).cuda(), 2.0**-6, 2.0**-7)
        acc0 = lf.acc.cpu().numpy()
        lf.step(3)
        p = np.concatenate([q[0] for q in parts]); a0 = np.concatenate([q[1] for q in parts])
        print(mode, "init_all==pos", np.array_equal(parts[0][2], pos), "init acc mismatch rows", int((a0 != acc0).any(1).sum()),
              "final pos mismatch rows", int((p != lf.pos.cpu().numpy()).any(1).sum()))
    dist.destroy_process_group()

if __name__ == "__main__":
    for mode in ("sync", "async"):
        s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
        mp.spawn(worker, args=(2, port, mode, None), nprocs=2, join=True)
