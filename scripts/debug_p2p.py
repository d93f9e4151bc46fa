import os, sys, socket
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch, torch.multiprocessing as mp
from test_distributed_gpu import _p2p_nbody_worker, _port
if __name__ == "__main__":
    for world in (2,):
        out = "/tmp/nb.npz"
        mp.spawn(_p2p_nbody_worker, args=(world, _port(), 8192, 3, out), nprocs=world, join=True)
        z = np.load(out)
        for a, b in (("p", "lp"), ("v", "lv"), ("a", "la"), ("allpos", "lp")):
            d = z[a] != z[b]
            rows = np.where(d.any(1))[0]
            print(a, b, "mismatch rows", len(rows), rows[:10], "max abs diff", np.abs(z[a]-z[b]).max())
