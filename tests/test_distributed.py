"""CPU, world_size 2-3 over gloo: the multi-GPU partitioning logic.

The compute backend is injected with the oracle (CPU) so the exchange logic --
shard offsets, in-place position all-gather, halo planes, global-boundary
clamps, interior/boundary split -- is exercised without a GPU. The property
checked is the one the design promises: sharded == unsharded, bit for bit.
"""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


class OracleNBodyKernels:
    """CPU stand-in for distributed.CudaNBodyKernels (same chunked structure)."""

    def __init__(self, chunk: int):
        import oracle

        self.o = oracle.Restatement()
        self.chunk = chunk

    def nchunks(self, nj):
        return (nj + self.chunk - 1) // self.chunk

    def partials(self, ipos, jpos, eps, out):
        self.o.calc_acc_partials(ipos.numpy(), jpos.numpy(), eps, self.chunk, out=out.numpy())

    def update(self, pos, vel, acc, partials, nchunks, h_end, h_begin, dt, phases):
        n = lambda t: t.numpy() if t is not None else None  # noqa: E731
        self.o.kdk_update(n(pos), n(vel), acc.numpy(), n(partials), nchunks, h_end, h_begin, dt, phases)


class OracleSlabKernels:
    """CPU stand-in for distributed.CudaSlabKernels: the oracle on the halo-extended slab."""

    def __init__(self, *args):
        import oracle

        self.o = oracle.Restatement()
        self.args = args

    def run2(self, f, fn):
        fn.numpy()[...] = self.o.diffusion_run(f.numpy(), 2, *self.args)
        return True

    def run2_planes(self, f, fn, p0, p1, p2=0, p3=0):
        if p1 > p0 or p3 > p2:
            out = self.o.diffusion_run(f.numpy(), 2, *self.args)
            fn.numpy()[p0:p1] = out[p0:p1]
            fn.numpy()[p2:p3] = out[p2:p3]
        return True

    def slab(self, f, fn, halo_lo, halo_hi, i_begin, i_end):
        a = f.numpy()
        lo = halo_lo.numpy() if halo_lo is not None else a[0]  # absent halo == clamp IMAX(i-1,0)
        hi = halo_hi.numpy() if halo_hi is not None else a[-1]
        ext = np.concatenate([lo[None], a, hi[None]], axis=0)
        out = self.o.diffusion3d(ext, *self.args)
        fn.numpy()[i_begin:i_end] = out[1 + i_begin:1 + i_end]


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _init(rank, world, port):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)


def _nbody_worker(rank, world, port, n, steps, out_path):
    _init(rank, world, port)
    from paper_2411_18889_b200.distributed import ShardedLeapfrog
    from paper_2411_18889_b200.nbody import plummer_numpy

    pos, vel = plummer_numpy(n, 21)
    nl = n // world
    sim = ShardedLeapfrog(torch.from_numpy(pos[rank * nl:(rank + 1) * nl]),
                          torch.from_numpy(vel[rank * nl:(rank + 1) * nl]), 2.0 ** -6, 2.0 ** -7,
                          kernels=OracleNBodyKernels(64))
    sim.step(steps)
    gp = [torch.empty_like(sim.pos) for _ in range(world)]
    gv = [torch.empty_like(sim.vel) for _ in range(world)]
    ga = [torch.empty_like(sim.acc) for _ in range(world)]
    dist.all_gather(gp, sim.pos.clone())
    dist.all_gather(gv, sim.vel)
    dist.all_gather(ga, sim.acc)
    if rank == 0:
        np.savez(out_path, pos=torch.cat(gp).numpy(), vel=torch.cat(gv).numpy(), acc=torch.cat(ga).numpy())
    dist.destroy_process_group()


def _diff_worker(rank, world, port, shape, steps, out_path):
    _init(rank, world, port)
    from paper_2411_18889_b200.distributed import SlabDiffusion

    f0 = np.random.default_rng(4).random(shape, dtype=np.float32)
    args = (0.1, 0.12, 0.09, 1e-3, 1.0)
    counts = [shape[0] // world + (1 if r < shape[0] % world else 0) for r in range(world)]
    lo = sum(counts[:rank])
    sim = SlabDiffusion(torch.from_numpy(f0[lo:lo + counts[rank]].copy()), *args, kernels=OracleSlabKernels(*args))
    sim.step(steps)
    parts = [None] * world
    dist.all_gather_object(parts, sim.f.numpy())
    if rank == 0:
        np.save(out_path, np.concatenate(parts, axis=0))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_sharded_leapfrog_equals_unsharded(tmp_path, world):
    n, steps = 512, 3
    out = tmp_path / "nbody.npz"
    mp.spawn(_nbody_worker, args=(world, _free_port(), n, steps, str(out)), nprocs=world, join=True)
    got = np.load(out)
    # unsharded: world 1 through the same class and kernels
    out1 = tmp_path / "nbody1.npz"
    mp.spawn(_nbody_worker, args=(1, _free_port(), n, steps, str(out1)), nprocs=1, join=True)
    want = np.load(out1)
    for k in ("pos", "vel", "acc"):
        assert np.array_equal(got[k].view(np.uint32), want[k].view(np.uint32)), k


def test_unsharded_chunked_leapfrog_tracks_reference_kdk(tmp_path):
    """The chunked structure stays within FP32 tolerance of the plain oracle KDK."""
    import oracle

    from paper_2411_18889_b200.nbody import plummer_numpy

    n, steps = 512, 3
    out1 = tmp_path / "nbody1.npz"
    mp.spawn(_nbody_worker, args=(1, _free_port(), n, steps, str(out1)), nprocs=1, join=True)
    got = np.load(out1)
    pos, vel = plummer_numpy(n, 21)
    wp, wv, wa = oracle.Restatement().leapfrog(pos, vel, 2.0 ** -6, 2.0 ** -7, steps)
    assert np.linalg.norm(got["pos"] - wp) / np.linalg.norm(wp) < 1e-6
    assert np.linalg.norm(got["acc"] - wa) / np.linalg.norm(wa) < 1e-5


@pytest.mark.parametrize("world,shape", [(2, (12, 9, 10)), (3, (10, 7, 8)), (2, (4, 5, 6))])
def test_slab_diffusion_equals_full_grid(tmp_path, world, shape):
    import oracle

    steps = 4
    out = tmp_path / "diff.npy"
    mp.spawn(_diff_worker, args=(world, _free_port(), shape, steps, str(out)), nprocs=world, join=True)
    got = np.load(out)
    f0 = np.random.default_rng(4).random(shape, dtype=np.float32)
    want = oracle.Restatement().diffusion_run(f0, steps, 0.1, 0.12, 0.09, 1e-3, 1.0)
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))


def test_shard_plan_requires_divisible_n():
    from paper_2411_18889_b200.distributed import ShardPlan

    p = ShardPlan(1 << 22, 8, 3)
    assert (p.n_local, p.lo, p.hi) == (1 << 19, 3 << 19, 4 << 19)


def _ckpt_nbody_worker(rank, world, port, n, ckpt, out_path):
    """4 steps straight vs 2 (left open: pending half-kick) + checkpoint + fresh driver + resume + 2."""
    _init(rank, world, port)
    from paper_2411_18889_b200 import checkpoint
    from paper_2411_18889_b200.distributed import ShardedLeapfrog
    from paper_2411_18889_b200.nbody import plummer_numpy

    pos, vel = plummer_numpy(n, 5)
    nl = n // world
    mk = lambda: ShardedLeapfrog(torch.from_numpy(pos[rank * nl:(rank + 1) * nl]),  # noqa: E731
                                 torch.from_numpy(vel[rank * nl:(rank + 1) * nl]), 2.0 ** -6, 2.0 ** -7,
                                 kernels=OracleNBodyKernels(64))
    a = mk()
    a.step(4)
    b = mk()
    b.step(2, close=False)
    checkpoint.save(b, ckpt)
    c = mk()
    checkpoint.load(c, ckpt)
    c.step(2)
    ok = all(np.array_equal(x.numpy().view(np.uint32), y.numpy().view(np.uint32))
             for x, y in ((a.pos, c.pos), (a.vel, c.vel), (a.acc, c.acc))) and c.steps == 4
    flags = [None] * world
    dist.all_gather_object(flags, ok)
    if rank == 0:
        np.save(out_path, np.array(flags))
    dist.destroy_process_group()


def _ckpt_diff_worker(rank, world, port, shape, ckpt, out_path):
    _init(rank, world, port)
    from paper_2411_18889_b200 import checkpoint
    from paper_2411_18889_b200.distributed import SlabDiffusion

    f0 = np.random.default_rng(8).random(shape, dtype=np.float32)
    args = (0.1, 0.12, 0.09, 1e-3, 1.0)
    nl = shape[0] // world
    mk = lambda: SlabDiffusion(torch.from_numpy(f0[rank * nl:(rank + 1) * nl].copy()), *args,  # noqa: E731
                               kernels=OracleSlabKernels(*args))
    a = mk()
    a.step(5)
    b = mk()
    b.step(3)
    checkpoint.save(b, ckpt)
    c = mk()
    checkpoint.load(c, ckpt)
    c.step(2)
    ok = np.array_equal(a.f.numpy().view(np.uint32), c.f.numpy().view(np.uint32)) and c.steps_done == 5
    flags = [None] * world
    dist.all_gather_object(flags, ok)
    if rank == 0:
        np.save(out_path, np.array(flags))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [1, 2])
def test_sharded_leapfrog_checkpoint_resume_bit_identical(tmp_path, world):
    out = tmp_path / "ok.npy"
    mp.spawn(_ckpt_nbody_worker, args=(world, _free_port(), 256, str(tmp_path / "nb.{rank}.pt"), str(out)),
             nprocs=world, join=True)
    assert np.load(out).all()
    assert sorted(p.name for p in tmp_path.glob("nb.*.pt")) == [f"nb.{r}.pt" for r in range(world)]


@pytest.mark.parametrize("world", [1, 2])
def test_slab_diffusion_checkpoint_resume_bit_identical(tmp_path, world):
    out = tmp_path / "ok.npy"
    mp.spawn(_ckpt_diff_worker, args=(world, _free_port(), (8, 6, 7), str(tmp_path / "df.{rank}.pt"), str(out)),
             nprocs=world, join=True)
    assert np.load(out).all()


def test_checkpoint_rejects_mismatched_run(tmp_path):
    """A shard checkpoint refuses to load into a different decomposition."""
    from paper_2411_18889_b200.distributed import ShardedLeapfrog

    sd = {"kind": "ShardedLeapfrog", "n_total": 512, "world": 2, "rank": 0}

    class Fake:
        plan = type("P", (), {"n_total": 256, "world": 1, "rank": 0})()
        eps, dt = 0.1, 0.1

    with pytest.raises(ValueError, match="checkpoint is for"):
        ShardedLeapfrog.load_state_dict(Fake(), sd)
    with pytest.raises(ValueError, match="not a ShardedLeapfrog"):
        ShardedLeapfrog.load_state_dict(Fake(), {"kind": "Leapfrog"})


def _random_cases_worker(rank, world, port, out_path):
    """Seeded random cases inside one process group (the reference's seeded property-test style,
    pkg/tests/test_acceptance.py:136-206): ragged slab splits, N not a power of two, runs left
    open and closed -- each compared bit for bit with the unsharded computation on rank 0."""
    _init(rank, world, port)
    import random

    import oracle
    from paper_2411_18889_b200.distributed import ShardedLeapfrog, SlabDiffusion
    from paper_2411_18889_b200.nbody import plummer_numpy

    o = oracle.Restatement()
    rnd = random.Random(987654321)
    ok = True
    for _ in range(6):  # n-body
        n = world * rnd.randint(8, 96)
        steps, chunk, close = rnd.randint(1, 4), rnd.choice([16, 64, 100]), rnd.random() < 0.5
        pos, vel = plummer_numpy(n, rnd.randint(0, 1000))
        nl = n // world
        sim = ShardedLeapfrog(torch.from_numpy(pos[rank * nl:(rank + 1) * nl]),
                              torch.from_numpy(vel[rank * nl:(rank + 1) * nl]), 2.0 ** -6, 2.0 ** -7,
                              kernels=OracleNBodyKernels(chunk))
        sim.step(steps, close=close)
        gp = [torch.empty_like(sim.pos) for _ in range(world)]
        gv = [torch.empty_like(sim.vel) for _ in range(world)]
        dist.all_gather(gp, sim.pos.clone())
        dist.all_gather(gv, sim.vel)
        if rank == 0:
            # unsharded, same chunked structure: init acc, open, (force, update) x steps
            p, v = pos.copy(), vel.copy()
            a = np.empty_like(p)
            nch = (n + chunk - 1) // chunk
            part = np.empty((nch * n, 4), np.float32)
            h = 0.5 * 2.0 ** -7
            o.calc_acc_partials(p, p, 2.0 ** -6, chunk, out=part)
            o.kdk_update(None, None, a, part, nch, 0.0, 0.0, 0.0, 1)
            o.kdk_update(p, v, a, None, nch, 0.0, h, 2.0 ** -7, 4)
            for s in range(steps):
                o.calc_acc_partials(p, p, 2.0 ** -6, chunk, out=part)
                last = close and s + 1 == steps
                o.kdk_update(p, v, a, part, nch, h, h, 2.0 ** -7, 1 | 2 | (0 if last else 4))
            ok &= np.array_equal(torch.cat(gp).numpy().view(np.uint32), p.view(np.uint32))
            ok &= np.array_equal(torch.cat(gv).numpy().view(np.uint32), v.view(np.uint32))
    for _ in range(6):  # diffusion, ragged slabs
        counts = [rnd.randint(2, 6) for _ in range(world)]
        shape = (sum(counts), rnd.randint(1, 7), rnd.randint(1, 9))
        steps = rnd.randint(1, 5)
        args = (0.11, 0.07, 0.13, 1e-3, 1.0)
        f0 = np.random.default_rng(rnd.randint(0, 1000)).random(shape, dtype=np.float32)
        lo = sum(counts[:rank])
        sim = SlabDiffusion(torch.from_numpy(f0[lo:lo + counts[rank]].copy()), *args,
                            kernels=OracleSlabKernels(*args))
        sim.step(steps)
        parts = [None] * world
        dist.all_gather_object(parts, sim.f.numpy())
        if rank == 0:
            want = o.diffusion_run(f0, steps, *args)
            ok &= np.array_equal(np.concatenate(parts, axis=0).view(np.uint32), want.view(np.uint32))
    if rank == 0:
        np.save(out_path, np.array([ok]))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_drivers_random_cases(tmp_path, world):
    out = tmp_path / "ok.npy"
    mp.spawn(_random_cases_worker, args=(world, _free_port(), str(out)), nprocs=world, join=True)
    assert np.load(out).all()


def _mismatch_worker(rank, world, port, out_path):
    _init(rank, world, port)
    from paper_2411_18889_b200.distributed import SlabDiffusion

    args = (0.1, 0.12, 0.09, 1e-3, 1.0)
    f = torch.zeros((3, 5, 8 if rank == 0 else 12))  # rank 1 holds wider planes
    try:
        SlabDiffusion(f, *args, kernels=OracleSlabKernels(*args))
        msg = "no error"
    except ValueError as e:
        msg = str(e)
    parts = [None] * world
    dist.all_gather_object(parts, msg)
    if rank == 0:
        np.save(out_path, np.array(parts))
    dist.destroy_process_group()


def test_slab_diffusion_rejects_mismatched_planes_on_every_rank(tmp_path):
    """A plane-shape mismatch raises ValueError on all ranks (checked collectively at setup)
    instead of one rank raising and the others deadlocking in the first halo exchange."""
    out = tmp_path / "m.npy"
    mp.spawn(_mismatch_worker, args=(2, _free_port(), str(out)), nprocs=2, join=True)
    msgs = np.load(out)
    assert all("different planes" in m for m in msgs), msgs


def _run2_worker(rank, world, port, counts, ny, nz, steps, out_path):
    _init(rank, world, port)
    from paper_2411_18889_b200.distributed import SlabDiffusion

    f0 = np.random.default_rng(6).random((sum(counts), ny, nz), dtype=np.float32)
    args = (0.1, 0.12, 0.09, 1e-3, 1.0)
    lo = sum(counts[:rank])
    sim = SlabDiffusion(torch.from_numpy(f0[lo:lo + counts[rank]].copy()), *args, kernels=OracleSlabKernels(*args))
    sim.run(steps[0])
    sim.step(1)          # the per-step path continues from run()'s state
    sim.run(steps[1])
    parts = [None] * world
    dist.all_gather_object(parts, (sim.f.numpy(), sim.steps_done))
    if rank == 0:
        np.save(out_path, np.concatenate([p[0] for p in parts], axis=0))
        assert all(p[1] == steps[0] + 1 + steps[1] for p in parts)
    dist.destroy_process_group()


@pytest.mark.parametrize("world,counts,steps", [(2, (3, 4), (4, 5)), (3, (2, 5, 3), (6, 2)), (4, (2, 2, 3, 2), (3, 4)),
                                               (2, (7, 9), (4, 5)), (3, (6, 8, 11), (6, 3))])
def test_slab_run_two_steps_per_exchange_equals_full_grid(tmp_path, world, counts, steps):
    """SlabDiffusion.run: two steps per exchange of two halo planes (uneven slabs, odd
    remainders, mixed with step(); slabs of >= 6 planes take the overlapped pass -- interior
    while the halo travels, then the planes next to it) == the full-grid oracle run, bit for bit."""
    import oracle

    out = tmp_path / "r.npy"
    ny, nz = 5, 7
    mp.spawn(_run2_worker, args=(world, _free_port(), counts, ny, nz, steps, str(out)), nprocs=world, join=True)
    f0 = np.random.default_rng(6).random((sum(counts), ny, nz), dtype=np.float32)
    want = oracle.Restatement().diffusion_run(f0, steps[0] + 1 + steps[1], 0.1, 0.12, 0.09, 1e-3, 1.0)
    assert np.array_equal(np.load(out).view(np.uint32), want.view(np.uint32))
