"""Randomised parity sweep (a longer, non-derandomised companion of tests/test_properties_gpu.py).

    python scripts/fuzz_parity.py [--cases N] [--seed S]

Random diffusion grids through Diffusion3D.run (every dispatch path: resident bricks,
cooperative multi-step, two steps per HBM pass with first-use plan timing, single-step
kernels) and random calc_acc sizes (exact and fast), each against the oracle restatement:
bit for bit for diffusion and exact n-body, relL2 < 1e-5 for fast n-body. Prints failures and
a summary; exit status 1 on any failure.
"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import oracle  # noqa: E402  (checker only)
import paper_2411_18889_b200 as b2  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", type=int, default=200)
    ap.add_argument("--seed", type=int, default=None)
    args = ap.parse_args()
    seed = args.seed if args.seed is not None else int.from_bytes(os.urandom(4), "little")
    rng = np.random.default_rng(seed)
    ref = oracle.Restatement()
    fails = 0
    for case in range(args.cases):
        if case % 2 == 0:
            nz = 4 * int(rng.integers(1, 300)) if rng.random() < 0.8 else int(rng.integers(1, 200))
            nx, ny = int(rng.integers(1, 80)), int(rng.integers(1, 80))
            if nx * ny * nz > 6_000_000:
                nx = max(1, 6_000_000 // (ny * nz))
            steps = int(rng.integers(0, 9))
            dargs = (0.031, 0.027, 0.022, 2e-5, 1.0)
            f0 = rng.random((nx, ny, nz), dtype=np.float32)
            want = ref.diffusion_run(f0, steps, *dargs)
            got = b2.Diffusion3D(torch.from_numpy(f0).cuda(), *dargs).run(steps).cpu().numpy()
            if not np.array_equal(got.view(np.uint32), want.view(np.uint32)):
                fails += 1
                print(f"FAIL diffusion {(nx, ny, nz)} steps={steps}", flush=True)
        else:
            ni, nj = int(rng.integers(1, 5000)), int(rng.integers(1, 20000))
            jpos = np.empty((nj, 4), np.float32)
            jpos[:, :3] = rng.uniform(-1, 1, (nj, 3))
            jpos[:, 3] = rng.uniform(0.5, 1.5, nj) / nj
            ipos = jpos[rng.integers(0, nj, ni)].copy()
            pot = bool(rng.random() < 0.3)
            want = ref.calc_acc(ipos, jpos, 2.0 ** -6, potential=pot)
            ip, jp = torch.from_numpy(ipos).cuda(), torch.from_numpy(jpos).cuda()
            out = torch.empty_like(ip)
            b2.calc_acc(ni, ip, out, nj, jp, 2.0 ** -6, potential=pot, exact=True)
            ex = out.cpu().numpy()
            b2.calc_acc(ni, ip, out, nj, jp, 2.0 ** -6, potential=pot)
            fa = out.cpu().numpy()
            rel = np.linalg.norm(fa[:, :3] - want[:, :3]) / max(np.linalg.norm(want[:, :3]), 1e-30)
            if not np.array_equal(ex.view(np.uint32), want.view(np.uint32)) or rel >= 1e-5:
                fails += 1
                print(f"FAIL calc_acc ni={ni} nj={nj} pot={pot} exact_eq={np.array_equal(ex, want)} rel={rel:.2e}",
                      flush=True)
    print(f"seed {seed}: {args.cases} cases, {fails} failures", flush=True)
    sys.exit(1 if fails else 0)


if __name__ == "__main__":
    main()
