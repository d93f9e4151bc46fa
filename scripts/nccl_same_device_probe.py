"""Probe: can NCCL run world > 1 with every rank on cuda:0 (one-GPU rehearsal of the N>1 path)?"""
import datetime
import os

import torch
import torch.distributed as dist

rank = int(os.environ["RANK"])
world = int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(0)
dist.init_process_group("nccl", timeout=datetime.timedelta(seconds=60), device_id=torch.device("cuda", 0))
x = torch.full((4,), float(rank), device="cuda")
out = torch.empty(4 * world, device="cuda")
try:
    dist.all_gather_into_tensor(out, x)
    torch.cuda.synchronize()
    print(f"rank {rank}: all_gather ok {out.tolist()}", flush=True)
except Exception as e:  # noqa: BLE001
    print(f"rank {rank}: all_gather failed: {type(e).__name__}: {e}", flush=True)
dist.destroy_process_group()
