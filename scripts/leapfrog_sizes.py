"""Leapfrog.step(k) device time across N (median of 5 fresh runs, host launch latency kept out
by a queued spin): interactions/s and the FP32 fraction at 20 flop/interaction.

    python scripts/leapfrog_sizes.py [n ...]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2411_18889_b200 as b2  # noqa: E402

PEAK = 74.2e12  # live FFMA2 probe
sizes = [int(x) for x in sys.argv[1:]] or [2048, 4096, 6144, 8192, 9472, 12288, 16384, 32768]
for n in sizes:
    pos, vel = b2.plummer(n, 42)
    steps = 16
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    runs = []
    for r in range(6):
        lf = b2.Leapfrog(pos.clone(), vel.clone(), 2.0 ** -6, 2.0 ** -7)
        lf.step(steps)  # graphs (mid N) captured on the first call
        torch.cuda.synchronize()
        torch.cuda._sleep(1_000_000)
        ev[0].record()
        lf.step(steps)
        ev[1].record()
        torch.cuda.synchronize()
        runs.append(ev[0].elapsed_time(ev[1]))
    ms = sorted(runs[1:])[2]
    gi = n * n * steps / (ms * 1e-3)
    print(json.dumps({"n": n, "us_per_step": round(ms * 1e3 / steps, 2), "ginter_s": round(gi / 1e9, 1),
                      "fp32_frac": round(20 * gi / PEAK, 4)}), flush=True)
