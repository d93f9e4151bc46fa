"""Randomised parity sweep (a longer, non-derandomised companion of tests/test_properties_gpu.py).

    python scripts/fuzz_parity.py [--cases N] [--seed S]

Random diffusion grids through Diffusion3D.run (every dispatch path: resident bricks,
cooperative multi-step, two steps per HBM pass with first-use plan timing, single-step
kernels) and random calc_acc sizes (exact and fast, incl. the in-kernel ring reduction past
~63k i), each against the oracle restatement: bit for bit for diffusion and exact n-body,
relL2 < 1e-5 for fast n-body. Round 2 adds: the persistent small-N leapfrog (random N up to
9472, steps, potential) against the two-kernel schedule built from the C ABI
(b2_calc_acc_partials + b2_kdk_update), bit for bit; and b2_diffusion3d_run2_planes over a
random split of the planes against the whole two-step pass, bit for bit. Prints failures
and a summary; exit status 1 on any failure.
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
        if case % 4 == 2:
            fails += leapfrog_case(rng)
            continue
        if case % 4 == 3:
            fails += planes_case(rng)
            continue
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
            if rng.random() < 0.1:  # past the partials workspace: the in-kernel ring reduction
                ni, nj = int(rng.integers(63_500, 90_000)), int(rng.integers(1, 3000))
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


def two_kernel_leapfrog(pos, vel, eps, dt, steps, potential):
    """The two-kernel KDK schedule from the C ABI: force partials + the fused update."""
    from paper_2411_18889_b200 import _lib

    lib, sh = _lib.load(), _lib.stream_handle()
    n = pos.shape[0]
    flags = _lib.B2_POTENTIAL if potential else 0
    nch = lib.b2_calc_acc_nchunks(n, flags)
    part = torch.empty((nch * n, 4), device="cuda")
    acc = torch.empty_like(pos)
    h = 0.5 * dt

    def force():
        assert lib.b2_calc_acc_partials(n, pos.data_ptr(), n, pos.data_ptr(), eps, flags, part.data_ptr(), sh) == 0

    force()
    assert lib.b2_kdk_update(n, None, None, acc.data_ptr(), part.data_ptr(), nch, 0.0, 0.0, 0.0, 1, sh) == 0
    if steps:
        assert lib.b2_kdk_update(n, pos.data_ptr(), vel.data_ptr(), acc.data_ptr(), None, 1, 0.0, h, dt, 4, sh) == 0
    for st in range(steps):
        force()
        ph = 1 | 2 | (0 if st + 1 == steps else 4)
        assert lib.b2_kdk_update(n, pos.data_ptr(), vel.data_ptr(), acc.data_ptr(), part.data_ptr(), nch, h, h, dt,
                                 ph, sh) == 0
    return pos, vel, acc


def leapfrog_case(rng) -> int:
    n, steps, pot = int(rng.integers(2, 9473)), int(rng.integers(0, 5)), bool(rng.random() < 0.3)
    pos, vel = b2.plummer_numpy(n, int(rng.integers(0, 2 ** 16)))
    lf = b2.Leapfrog(torch.from_numpy(pos).cuda(), torch.from_numpy(vel).cuda(), 2.0 ** -6, 2.0 ** -7, potential=pot)
    lf.step(steps)
    p, v, a = two_kernel_leapfrog(torch.from_numpy(pos).cuda(), torch.from_numpy(vel).cuda(), 2.0 ** -6, 2.0 ** -7,
                                  steps, pot)
    ok = all(torch.equal(x.view(torch.int32), y.view(torch.int32)) for x, y in ((lf.pos, p), (lf.vel, v), (lf.acc, a)))
    if not ok:
        print(f"FAIL leapfrog n={n} steps={steps} pot={pot}", flush=True)
    return 0 if ok else 1


def planes_case(rng) -> int:
    from paper_2411_18889_b200.distributed import CudaSlabKernels

    nz = 128 * int(rng.integers(1, 9))
    nx, ny = int(rng.integers(2, 40)), int(rng.integers(1, 40))
    args = (0.031, 0.027, 0.022, 2e-5, 1.0)
    f = torch.rand((nx, ny, nz), device="cuda")
    k = CudaSlabKernels(*args)
    if not k.run2_planes(f, torch.empty_like(f), 0, 0):
        return 0  # no two-steps-per-pass plan for this shape
    want = b2.Diffusion3D(f.clone(), *args).run(2)
    cuts = sorted(set(int(c) for c in rng.integers(0, nx + 1, 3)) | {0, nx})
    fn = torch.full_like(f, float("nan"))
    pieces = list(zip(cuts[:-1], cuts[1:]))
    rng.shuffle(pieces)
    while pieces:  # one or two ranges per call
        a = pieces.pop()
        b = pieces.pop() if pieces and rng.random() < 0.5 else (0, 0)
        assert k.run2_planes(f, fn, *a, *b)
    ok = torch.equal(fn.view(torch.int32), want.view(torch.int32))
    if not ok:
        print(f"FAIL run2_planes {(nx, ny, nz)} cuts={cuts}", flush=True)
    return 0 if ok else 1


if __name__ == "__main__":
    main()
