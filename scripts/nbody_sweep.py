"""Leapfrog throughput across N (which path each N takes: persistent small-N or two kernels per step)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2411_18889_b200 as b2  # noqa: E402

for n in [int(x) for x in (sys.argv[1:] or "1024 2048 4096 4736 6144 8192 16384 32768 65536 131072 262144".split())]:
    pos, vel = b2.plummer(n, 1)
    lf = b2.Leapfrog(pos, vel, 2.0 ** -6, 2.0 ** -7)
    steps = max(2, min(64, int(4e11 / n / n)))
    lf.step(2)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    lf.step(steps)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    print(f"N={n:7d}  {ms * 1e3:9.1f} us/step  {n * n / (ms * 1e-3) / 1e9:8.1f} Ginter/s", flush=True)
