"""Throughput across problem sizes on one GPU (evidence for DESIGN.md §7's size table).

    python scripts/perf_sweep.py [--out FILE]

N-body: Leapfrog.step (force + fused update per step; the persistent one-launch path below
32 x SMs particles) in interactions/s, and the fraction of the FP32 peak at 20 flop per
interaction. Diffusion: one reference-signature step (b2.diffusion3d) and the device-resident
run (Diffusion3D.run: resident bricks, cooperative multi-step or two steps per HBM pass,
whichever the planner takes) in GLUPS. CUDA-event timing after warm-up; inputs per size.
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2411_18889_b200 as b2  # noqa: E402

FP32_PEAK_TF = 74.2  # measured live by csrc/probe.cu on the round-1 boxes


def timed(fn, reps):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    fn()
    torch.cuda.synchronize()
    ev[0].record()
    for _ in range(reps):
        fn()
    ev[1].record()
    torch.cuda.synchronize()
    return ev[0].elapsed_time(ev[1]) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    rows = []
    for e in range(12, 22):
        n = 1 << e
        pos, vel = b2.plummer(n, 42)
        lf = b2.Leapfrog(pos, vel, 2.0 ** -6, 2.0 ** -7)
        steps = 16 if n <= 4736 else max(1, min(16, (1 << 34) // (n * n)))
        ms = timed(lambda: lf.step(steps), 2) / steps
        inter = float(n) * n / (ms * 1e-3)
        rows.append({"kind": "nbody Leapfrog.step", "n": n, "us_per_step": ms * 1e3, "ginter_s": inter / 1e9,
                     "fp32_frac": 20 * inter / 1e12 / FP32_PEAK_TF})
        print(json.dumps(rows[-1]), flush=True)
    for g in (64, 128, 256, 384, 512, 768, 1024):
        f = b2.init_grid(g, g, g, seed=7)
        fn = torch.empty_like(f)
        d = 1.0 / g
        dargs = (d, d, d, 0.1 * d * d, 1.0)
        cells = float(g) ** 3
        ms1 = timed(lambda: b2.diffusion3d(g, g, g, *dargs, f, fn), 10 if g <= 512 else 4)
        sim = b2.Diffusion3D(f.clone(), *dargs)
        nrun = 100 if g <= 256 else 20
        sim.run(4)  # first run of the shape: plan choice
        msr = timed(lambda: sim.run(nrun), 2) / nrun
        rows.append({"kind": "diffusion", "grid": g, "step_us": ms1 * 1e3, "step_glups": cells / (ms1 * 1e-3) / 1e9,
                     "step_hbm_frac": 8 * cells / (ms1 * 1e-3) / 6.65e12,
                     "run_us_per_step": msr * 1e3, "run_glups": cells / (msr * 1e-3) / 1e9})
        print(json.dumps(rows[-1]), flush=True)
        del f, fn, sim
        torch.cuda.empty_cache()
    if args.out:
        with open(args.out, "w") as fh:
            for r in rows:
                fh.write(json.dumps(r) + "\n")


if __name__ == "__main__":
    main()
