"""Run BASELINE configs[0] (N=4096 Plummer, 16 KDK steps) and configs[1] (128^3 x 100 steps) on
the GPU paths only -- a profiling target (ncu) and a quick timer for the small-grid kernels.

    python scripts/small_configs.py [--reps R]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2411_18889_b200 as b2  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--which", default="01")
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    if "0" in args.which:
        pos, vel = b2.plummer_numpy(4096, 42)
        for r in range(args.reps):
            lf = b2.Leapfrog(torch.from_numpy(pos).to(dev), torch.from_numpy(vel).to(dev), 2.0 ** -6, 2.0 ** -7)
            torch.cuda.synchronize()
            torch.cuda._sleep(1_000_000)  # host launch latency out of the events
            ev[0].record()
            lf.step(16)
            ev[1].record()
            torch.cuda.synchronize()
            ms = ev[0].elapsed_time(ev[1])
            print(f"configs[0] rep {r}: {ms * 1e3 / 16:.1f} us/step  {4096 ** 2 * 16 / (ms * 1e-3) / 1e9:.1f} Ginter/s")
    if "1" in args.which:
        g = 128
        dx = 1.0 / g
        f0 = b2.init_grid(g, g, g, seed=7, device=dev)
        for r in range(args.reps):
            sim = b2.Diffusion3D(f0.clone(), dx, dx, dx, 0.1 * dx * dx, 1.0)
            torch.cuda.synchronize()
            ev[0].record()
            sim.run(100)
            ev[1].record()
            torch.cuda.synchronize()
            ms = ev[0].elapsed_time(ev[1])
            print(f"configs[1] rep {r}: {ms * 1e3 / 100:.2f} us/step  {g ** 3 * 100 / (ms * 1e-3) / 1e9:.1f} GLUPS")


if __name__ == "__main__":
    main()
