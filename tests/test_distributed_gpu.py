"""GPU: the distributed classes on the CUDA kernels through NCCL (world_size 1 on the one
GPU gpurun gives; the multi-rank exchange logic is covered on CPU by test_distributed.py).

Checks that the sharded driver (NCCL in-place all-gather + partials + fused update) and
the slab driver (comm stream, interior/boundary split) reproduce the single-device
paths bit for bit.
"""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, port, out):
    import torch.distributed as dist

    import paper_2411_18889_b200 as b2
    from paper_2411_18889_b200.distributed import ShardedLeapfrog, SlabDiffusion

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    n, eps, dt = 8192, 2.0 ** -6, 2.0 ** -7
    pos, vel = b2.plummer(n, 42)
    sh = ShardedLeapfrog(pos, vel, eps, dt)
    sh.step(4)
    lf = b2.Leapfrog(pos.clone(), vel.clone(), eps, dt)
    lf.step(4)
    f = b2.init_grid(16, 24, 32, seed=2)
    sd = SlabDiffusion(f, 0.1, 0.1, 0.1, 1e-3, 1.0)
    sd.step(3)
    sd.run(5)  # two steps per exchange (world 1: the pass alone)
    ref = b2.Diffusion3D(f.clone(), 0.1, 0.1, 0.1, 1e-3, 1.0)
    ref.run(8)
    torch.cuda.synchronize()
    np.savez(out, sp=sh.pos.cpu().numpy(), sv=sh.vel.cpu().numpy(), sa=sh.acc.cpu().numpy(),
             lp=lf.pos.cpu().numpy(), lv=lf.vel.cpu().numpy(), la=lf.acc.cpu().numpy(),
             sd=sd.f.cpu().numpy(), rd=ref.field.cpu().numpy())
    dist.destroy_process_group()


def test_distributed_drivers_match_single_device(tmp_path):
    import torch.multiprocessing as mp

    out = tmp_path / "o.npz"
    mp.spawn(_worker, args=(_port(), str(out)), nprocs=1, join=True)
    z = np.load(out)
    for a, b in (("sp", "lp"), ("sv", "lv"), ("sa", "la"), ("sd", "rd")):
        assert np.array_equal(z[a].view(np.uint32), z[b].view(np.uint32)), a


def _p2p_worker(rank, world, port, shape, steps, out, lag=0.0):
    import time

    import torch.distributed as dist

    import paper_2411_18889_b200 as b2
    from paper_2411_18889_b200.distributed import SlabDiffusion

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    f0 = torch.from_numpy(np.random.default_rng(5).random(shape, dtype=np.float32))
    counts = [shape[0] // world + (1 if r < shape[0] % world else 0) for r in range(world)]
    lo = sum(counts[:rank])
    args = (0.1, 0.12, 0.09, 1e-3, 1.0)
    sim = SlabDiffusion(f0[lo:lo + counts[rank]].contiguous().cuda(), *args, transport="p2p")
    if lag:  # the last rank enqueues late every step: its neighbour's edge kernel must wait in the GPU
        for _ in range(steps):
            if rank == world - 1:
                time.sleep(lag)
            sim.step(1)
    else:
        sim.step(steps)
    torch.cuda.synchronize()
    parts = [None] * world
    dist.all_gather_object(parts, sim.f.cpu().numpy())
    sim.close()
    try:  # the peer mappings are gone: stepping must refuse, not touch unmapped memory
        sim.step(1)
        raise AssertionError("step after close did not raise")
    except RuntimeError:
        pass
    if rank == 0:
        ref = b2.Diffusion3D(f0.cuda(), *args)
        ref.run(steps)
        np.savez(out, got=np.concatenate(parts, axis=0), want=ref.field.cpu().numpy())
    dist.destroy_process_group()


@pytest.mark.parametrize("world,shape,steps", [(2, (24, 40, 64), 5), (3, (10, 7, 36), 4), (4, (17, 33, 128), 7),
                                               (2, (6, 9, 1024), 3)])
def test_p2p_fused_halo_slabs_match_full_grid(tmp_path, world, shape, steps):
    """transport='p2p': the edge-plane kernel pushes its rows, as tagged 16-byte words, into the
    neighbours' mailboxes (CUDA IPC) and polls its own -- no collective, event or host barrier per
    step -- bit-identical to the single-device run. Several processes share the one GPU here; on
    a multi-GPU box the same mapping goes over NVLink."""
    import torch.multiprocessing as mp

    out = tmp_path / "p2p.npz"
    mp.spawn(_p2p_worker, args=(world, _port(), shape, steps, str(out)), nprocs=world, join=True)
    z = np.load(out)
    assert np.array_equal(z["got"].view(np.uint32), z["want"].view(np.uint32))


def test_p2p_halo_waits_for_a_late_neighbour(tmp_path):
    """The halo has no host barrier: when one rank enqueues each step 0.3 s late, its
    neighbour's edge kernel polls its mailbox until the rows arrive (well inside the poll
    timeout) and the result is still bit-identical."""
    import torch.multiprocessing as mp

    out = tmp_path / "lag.npz"
    mp.spawn(_p2p_worker, args=(2, _port(), (12, 20, 64), 4, str(out), 0.3), nprocs=2, join=True)
    z = np.load(out)
    assert np.array_equal(z["got"].view(np.uint32), z["want"].view(np.uint32))


def _p2p_random_worker(rank, world, port, out):
    import torch.distributed as dist

    import paper_2411_18889_b200 as b2
    from paper_2411_18889_b200.distributed import SlabDiffusion

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(2024)  # same cases on every rank
    ok = []
    for _ in range(8):
        counts = [int(c) for c in rng.integers(2, 7, world)]  # uneven slabs, >= 2 planes each
        ny, nz, steps = int(rng.integers(1, 40)), 4 * int(rng.integers(1, 80)), int(rng.integers(1, 7))
        shape = (sum(counts), ny, nz)
        f0 = rng.random(shape, dtype=np.float32)
        args = (0.03, 0.025, 0.02, 2e-5, 1.0)
        lo = sum(counts[:rank])
        sim = SlabDiffusion(torch.from_numpy(f0[lo:lo + counts[rank]]).cuda(), *args, transport="p2p")
        sim.step(steps)
        torch.cuda.synchronize()
        parts = [None] * world
        dist.all_gather_object(parts, sim.f.cpu().numpy())
        sim.close()
        if rank == 0:
            want = b2.Diffusion3D(torch.from_numpy(f0).cuda(), *args).run(steps).cpu().numpy()
            got = np.concatenate(parts, axis=0)
            ok.append((shape, steps, bool(np.array_equal(got.view(np.uint32), want.view(np.uint32)))))
    if rank == 0:
        np.save(out, np.array([c[2] for c in ok]))
        print(ok)
    dist.destroy_process_group()


def test_p2p_halo_random_slabs(tmp_path):
    """Seeded random decompositions (uneven slabs of 2-6 planes, ny 1-39, nz 4-316, 1-6 steps)
    through the fused p2p halo, each bit-identical to the single-device run."""
    import torch.multiprocessing as mp

    out = tmp_path / "rand.npy"
    mp.spawn(_p2p_random_worker, args=(3, _port(), str(out)), nprocs=3, join=True)
    assert np.load(out).all()


def _p2p_run_worker(rank, world, port, counts, ny, nz, steps, out, lag=0.0):
    import time

    import torch.distributed as dist

    import paper_2411_18889_b200 as b2
    from paper_2411_18889_b200.distributed import SlabDiffusion

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    f0 = np.random.default_rng(12).random((sum(counts), ny, nz), dtype=np.float32)
    args = (0.03, 0.025, 0.02, 2e-5, 1.0)
    lo = sum(counts[:rank])
    sim = SlabDiffusion(torch.from_numpy(f0[lo:lo + counts[rank]]).cuda(), *args, transport="p2p")
    if lag:  # the last rank enqueues every exchange late: its neighbours' ingest waits in the GPU
        for _ in range(steps[0] // 2):
            if rank == world - 1:
                time.sleep(lag)
            sim.run(2)
        steps = (steps[0] // 2 * 2, steps[1])
    else:
        sim.run(steps[0])
    sim.step(1)  # the per-step fused halo resumes from run()'s state
    sim.run(steps[1])
    torch.cuda.synchronize()
    parts = [None] * world
    dist.all_gather_object(parts, sim.f.cpu().numpy())
    sim.close()
    if rank == 0:
        want = b2.Diffusion3D(torch.from_numpy(f0).cuda(), *args).run(steps[0] + 1 + steps[1]).cpu().numpy()
        np.savez(out, got=np.concatenate(parts, axis=0), want=want)
    dist.destroy_process_group()


@pytest.mark.parametrize("world,counts,ny,nz,steps", [(2, (3, 5), 20, 64, (4, 3)), (3, (2, 4, 3), 9, 1024, (6, 2)),
                                                      (4, (9, 7, 8, 8), 40, 128, (5, 6)),
                                                      (2, (12, 10), 24, 256, (6, 3)), (3, (6, 16, 7), 33, 512, (4, 5))])
def test_p2p_run_two_steps_per_exchange(tmp_path, world, counts, ny, nz, steps):
    """SlabDiffusion.run over the p2p transport: two-plane halos through peer-memory mailboxes
    (b2_diffusion3d_slab_halo2) every two steps, mixed with step(); slabs of >= 6 planes overlap
    the push with the planes that need no halo (b2_diffusion3d_run2_planes); bit-identical."""
    import torch.multiprocessing as mp

    out = tmp_path / "run2.npz"
    mp.spawn(_p2p_run_worker, args=(world, _port(), counts, ny, nz, steps, str(out)), nprocs=world, join=True)
    z = np.load(out)
    assert np.array_equal(z["got"].view(np.uint32), z["want"].view(np.uint32))


def test_p2p_run_waits_for_a_late_neighbour(tmp_path):
    """run()'s two-plane exchange has no host barrier: a rank that enqueues each exchange 0.3 s
    late makes its neighbour's ingest launch wait in the GPU; the result stays bit-identical."""
    import torch.multiprocessing as mp

    out = tmp_path / "runlag.npz"
    mp.spawn(_p2p_run_worker, args=(2, _port(), (4, 5), 12, 64, (6, 2), str(out), 0.3), nprocs=2, join=True)
    z = np.load(out)
    assert np.array_equal(z["got"].view(np.uint32), z["want"].view(np.uint32))
    out = tmp_path / "runlag2.npz"  # the overlapped pass (slabs of >= 6 planes)
    mp.spawn(_p2p_run_worker, args=(2, _port(), (8, 9), 12, 128, (6, 2), str(out), 0.3), nprocs=2, join=True)
    z = np.load(out)
    assert np.array_equal(z["got"].view(np.uint32), z["want"].view(np.uint32))


def _p2p_nbody_worker(rank, world, port, n, steps, out):
    import torch.distributed as dist

    import paper_2411_18889_b200 as b2
    from paper_2411_18889_b200.distributed import ShardedLeapfrog

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    pos, vel = b2.plummer_numpy(n, 8)
    nl = n // world
    sim = ShardedLeapfrog(torch.from_numpy(pos[rank * nl:(rank + 1) * nl]).cuda(),
                          torch.from_numpy(vel[rank * nl:(rank + 1) * nl]).cuda(), 2.0 ** -6, 2.0 ** -7,
                          transport="p2p")
    sim.step(steps)
    sim.step(2)  # re-open after a closed step
    torch.cuda.synchronize()
    parts = [None] * world
    dist.all_gather_object(parts, (sim.pos.cpu().numpy(), sim.vel.cpu().numpy(), sim.acc.cpu().numpy()))
    allpos = sim.pos_all.cpu().numpy()
    sim.close()
    try:
        sim.step(1)
        raise AssertionError("step after close did not raise")
    except RuntimeError:
        pass
    if rank == 0:
        lf = b2.Leapfrog(torch.from_numpy(pos).cuda(), torch.from_numpy(vel).cuda(), 2.0 ** -6, 2.0 ** -7)
        lf.step(steps)
        lf.step(2)
        np.savez(out, p=np.concatenate([q[0] for q in parts]), v=np.concatenate([q[1] for q in parts]),
                 a=np.concatenate([q[2] for q in parts]), allpos=allpos,
                 lp=lf.pos.cpu().numpy(), lv=lf.vel.cpu().numpy(), la=lf.acc.cpu().numpy())
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_p2p_fused_allgather_leapfrog_matches_single_device(tmp_path, world):
    """transport='p2p': the update kernel publishes positions into every peer's buffer (CUDA IPC);
    sharded KDK == single-device KDK, bit for bit, and every rank's pos_all is complete."""
    import torch.multiprocessing as mp

    out = tmp_path / "nb.npz"
    mp.spawn(_p2p_nbody_worker, args=(world, _port(), 8192, 3, str(out)), nprocs=world, join=True)
    z = np.load(out)
    for a, b in (("p", "lp"), ("v", "lv"), ("a", "la"), ("allpos", "lp")):
        assert np.array_equal(z[a].view(np.uint32), z[b].view(np.uint32)), a


def test_bench_n_ranks_path_on_one_gpu(tmp_path):
    """bench.py's N > 1 path end to end (torchrun, i-shards with the fused position publish,
    i-slabs with peer-memory halos, max-over-ranks timing, one JSON line from rank 0) with two
    ranks sharing the one GPU (--same-device: gloo control plane). Not a scaling number."""
    import json
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(_port()), "bench.py", "--gpus", "2", "--same-device", "--steps", "2",
           "--warmup", "3", "--particles", "65536", "--grid", "128", "--dsteps", "4"]
    out = subprocess.run(cmd, cwd=root, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    line = [ln for ln in out.stdout.splitlines() if ln.strip()]
    assert len(line) == 1, out.stdout[-2000:]  # stdout is the JSON line and nothing else
    assert len(line[0]) < 2600  # the driver keeps ~3000 characters of the tail
    d = json.loads(line[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and "i-shard x2" in d["config"]["parallelism"]
    assert d["scaling"] == "strong" and "scale_anchor" in d["config"]["scaling_note"]
    dif = d["secondary"]["diffusion"]
    assert dif["value"] > 0 and "slabs" in dif["what"] and dif["bit_identical"]
    assert d["parity"]["ok"] and d["parity"]["shard_eq_unsharded"]
    assert d["e2e"]["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] == 16 * 65536
    run = d["secondary"]["diffusion_run"]
    assert run["value"] > 0 and run["bit_identical"]
    anchor = d["secondary"]["scale_anchor"]  # the same N / grid on one GPU
    assert anchor["nbody"]["n"] == 65536 and anchor["nbody"]["value"] > 0
    assert anchor["diffusion_step"]["grid"] == 128 and anchor["diffusion_run"]["value"] > 0


def _p2p_ckpt_worker(rank, world, port, ckpt, out):
    import torch.distributed as dist

    from paper_2411_18889_b200 import checkpoint
    from paper_2411_18889_b200.distributed import SlabDiffusion

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    shape, args = (12, 20, 64), (0.1, 0.12, 0.09, 1e-3, 1.0)
    f0 = torch.from_numpy(np.random.default_rng(8).random(shape, dtype=np.float32))
    nl = shape[0] // world
    mk = lambda: SlabDiffusion(f0[rank * nl:(rank + 1) * nl].contiguous().cuda(), *args,  # noqa: E731
                               transport="p2p")
    a = mk()
    a.step(5)
    b = mk()
    b.step(3)
    checkpoint.save(b, ckpt)
    c = mk()
    checkpoint.load(c, ckpt)
    c.step(2)
    torch.cuda.synchronize()
    ok = bool(np.array_equal(a.f.cpu().numpy().view(np.uint32), c.f.cpu().numpy().view(np.uint32)))
    flags = [None] * world
    dist.all_gather_object(flags, ok)
    for s in (a, b, c):
        s.close()
    if rank == 0:
        np.save(out, np.array(flags))
    dist.destroy_process_group()


def test_p2p_slab_checkpoint_resume_bit_identical(tmp_path):
    """Resuming the p2p slab transport restarts the mailbox exchange at the loaded state."""
    import torch.multiprocessing as mp

    out = tmp_path / "ok.npy"
    mp.spawn(_p2p_ckpt_worker, args=(2, _port(), str(tmp_path / "s.{rank}.pt"), str(out)), nprocs=2, join=True)
    assert np.load(out).all()


def _nvls_worker(rank, world, port, n, steps, out):
    import torch.distributed as dist

    import paper_2411_18889_b200 as b2
    from paper_2411_18889_b200 import _lib
    from paper_2411_18889_b200.distributed import ShardedLeapfrog

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    pos, vel = b2.plummer_numpy(n, 8)
    nl = n // world
    mk = lambda: ShardedLeapfrog(torch.from_numpy(pos[rank * nl:(rank + 1) * nl]).cuda(),  # noqa: E731
                                 torch.from_numpy(vel[rank * nl:(rank + 1) * nl]).cuda(), 2.0 ** -6, 2.0 ** -7,
                                 transport="nvls")
    res = {}
    try:
        sim = mk()
    except _lib.SolomonError as e:  # every rank must see the same verdict (no one left in a collective)
        res["error"] = str(e)
    else:
        sim.step(steps)
        sim.step(2)  # re-open after a closed step
        torch.cuda.synchronize()
        res.update(p=sim.pos.cpu().numpy(), v=sim.vel.cpu().numpy(), a=sim.acc.cpu().numpy(),
                   allpos=sim.pos_all.cpu().numpy())
        sim.close()
        res["after_close"] = sim.pos_all.cpu().numpy()  # the state stays readable once unmapped
        try:
            sim.step(1)
            res["error"] = "step after close did not raise"
        except RuntimeError:
            pass
    parts = [None] * world
    dist.all_gather_object(parts, res)
    if rank == 0:
        lf = b2.Leapfrog(torch.from_numpy(pos).cuda(), torch.from_numpy(vel).cuda(), 2.0 ** -6, 2.0 ** -7)
        lf.step(steps)
        lf.step(2)
        np.savez(out, errors=np.array([q.get("error", "") for q in parts]),
                 lp=lf.pos.cpu().numpy(), lv=lf.vel.cpu().numpy(), la=lf.acc.cpu().numpy(),
                 **({k: np.concatenate([q[k] for q in parts]) for k in ("p", "v", "a")}
                    if all("p" in q for q in parts) else {}),
                 **({"allpos": parts[0]["allpos"], "after_close": parts[0]["after_close"]} if "allpos" in parts[0]
                    else {}))
    dist.destroy_process_group()


def test_nvls_multicast_allgather_leapfrog_matches_single_device(tmp_path):
    """transport='nvls' (NVSwitch multicast, b2_mc_*): the update kernel stores each position
    once through the multicast view and it lands in every rank's buffer. World 1 on the one
    GPU: the whole path (create, add, bind, multimem stores, release) against Leapfrog, bit
    for bit; skipped where the GPU has no multicast support."""
    import torch.multiprocessing as mp

    from paper_2411_18889_b200 import _lib

    if not _lib.load().b2_mc_supported(0):
        pytest.skip("no NVLS multicast object can be created here (GPU or fabric access)")
    out = tmp_path / "nvls.npz"
    mp.spawn(_nvls_worker, args=(1, _port(), 8192, 3, str(out)), nprocs=1, join=True)
    z = np.load(out)
    assert not any(z["errors"]), z["errors"]
    for a, b in (("p", "lp"), ("v", "lv"), ("a", "la"), ("allpos", "lp"), ("after_close", "lp")):
        assert np.array_equal(z[a].view(np.uint32), z[b].view(np.uint32)), a


def test_nvls_unavailable_fails_cleanly_on_every_rank(tmp_path):
    """Where no multicast object can be made -- two ranks on the same GPU, or a process that
    does not reach the NVSwitch fabric (this container) -- every rank gets the same
    SolomonError from the constructor (agreed collectively); none hangs."""
    import torch.multiprocessing as mp

    from paper_2411_18889_b200 import _lib

    worlds = [2] if _lib.load().b2_mc_supported(0) else [1, 2]
    for world in worlds:
        out = tmp_path / f"nvls{world}.npz"
        mp.spawn(_nvls_worker, args=(world, _port(), 8192, 1, str(out)), nprocs=world, join=True)
        errs = np.load(out)["errors"]
        assert len(errs) == world and all("nvls transport unavailable" in e for e in errs), errs
