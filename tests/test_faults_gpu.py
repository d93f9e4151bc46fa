"""GPU: failure detection of the device-side waits (DESIGN.md §6 "Failure detection").

A polling kernel whose data never arrives must neither hang the GPU nor kill the CUDA
context (round 1 trapped after a hard-coded 4 s): it gives up after the configurable poll
timeout, the host sees SolomonError, and the same process keeps computing correct results.
"""
from __future__ import annotations

import ctypes
import os
import socket
import time

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture
def short_timeout():
    from paper_2411_18889_b200 import _lib

    lib = _lib.load()
    old = lib.b2_poll_timeout_ms()
    _lib.set_poll_timeout(0.25)
    yield
    lib.b2_set_poll_timeout_ms(old)


def _context_still_works(restatement):
    import paper_2411_18889_b200 as b2

    f0 = np.random.default_rng(3).random((9, 10, 16), dtype=np.float32)
    args = (0.1, 0.1, 0.1, 1e-3, 1.0)
    f = torch.from_numpy(f0).cuda()
    fn = torch.empty_like(f)
    b2.diffusion3d(9, 10, 16, *args, f, fn)
    torch.cuda.synchronize()
    assert np.array_equal(fn.cpu().numpy().view(np.uint32), restatement.diffusion3d(f0, *args).view(np.uint32))


def test_poll_timeout_is_configurable():
    from paper_2411_18889_b200 import _lib

    lib = _lib.load()
    old = lib.b2_poll_timeout_ms()
    assert old >= 60_000  # default well above any healthy host stall (>= 60 s)
    _lib.set_poll_timeout(2.5)
    assert lib.b2_poll_timeout_ms() == 2500
    assert lib.b2_set_poll_timeout_ms(0) == _lib.B2_EINVAL
    lib.b2_set_poll_timeout_ms(old)


def test_expired_halo_poll_raises_and_context_survives(short_timeout, restatement):
    """An edge kernel waiting on a neighbour that never pushes: SolomonError naming the
    kernel, within ~the timeout; the fault is cleared and the context keeps working."""
    from paper_2411_18889_b200 import _lib

    lib = _lib.load()
    nxl, ny, nz = 4, 6, 16
    f = torch.rand((nxl, ny, nz), device="cuda")
    fn = torch.empty_like(f)
    mbox = torch.zeros(int(lib.b2_diffusion3d_mailbox_bytes(ny, nz)), dtype=torch.uint8, device="cuda")
    t0 = time.time()
    rc = lib.b2_diffusion3d_slab_edges(nxl, ny, nz, 0.1, 0.1, 0.1, 1e-3, 1.0, f.data_ptr(), fn.data_ptr(),
                                       mbox.data_ptr(), None, None, None, 0, 0, _lib.stream_handle())
    assert rc == 0
    with pytest.raises(_lib.SolomonError, match="k_diffusion_slab_edges"):
        _lib.check_fault(what="edge kernel")
    assert time.time() - t0 < 30
    _lib.check_fault()  # cleared: no error any more
    _context_still_works(restatement)


def test_expired_two_plane_ingest_raises_and_context_survives(short_timeout, restatement):
    from paper_2411_18889_b200 import _lib

    lib = _lib.load()
    nxl, ny, nz = 4, 5, 12
    f = torch.rand((nxl + 2, ny, nz), device="cuda")  # [2 halo | 4 own], no neighbour above
    mbox = torch.zeros(int(lib.b2_diffusion3d_mailbox2_bytes(ny, nz)), dtype=torch.uint8, device="cuda")
    assert lib.b2_diffusion3d_slab_halo2(nxl + 2, ny, nz, 2, nxl, f.data_ptr(), mbox.data_ptr(), None, None, None,
                                         0, 1, _lib.stream_handle()) == 0
    with pytest.raises(_lib.SolomonError, match="k_diffusion_slab_halo2"):
        _lib.check_fault()
    _context_still_works(restatement)


def test_expired_leapfrog_exchange_raises_and_context_survives(short_timeout):
    """The persistent small-N leapfrog with one CTA that never announces its positions
    (b2_debug_withhold_publish): the other CTAs' waits expire, Leapfrog.synchronize raises
    SolomonError naming the kernel, and the next run on the same context is exact again."""
    import paper_2411_18889_b200 as b2
    from paper_2411_18889_b200 import _lib

    lib = _lib.load()
    pos, vel = b2.plummer(4096, 9)
    try:
        lib.b2_debug_withhold_publish(3)
        lf = b2.Leapfrog(pos.clone(), vel.clone(), 2.0 ** -6, 2.0 ** -7)
        lf.step(2)
        with pytest.raises(_lib.SolomonError, match="k_leapfrog_small"):
            lf.synchronize()
    finally:
        lib.b2_debug_withhold_publish(-1)
    _lib.check_fault()  # cleared
    a = b2.Leapfrog(pos.clone(), vel.clone(), 2.0 ** -6, 2.0 ** -7)
    a.step(2)
    b = b2.Leapfrog(pos.clone(), vel.clone(), 2.0 ** -6, 2.0 ** -7, graphs=False)
    b.step(2)
    torch.cuda.synchronize()
    assert torch.equal(a.pos, b.pos) and torch.isfinite(a.pos).all()


def test_fault_word_is_sticky_until_cleared(short_timeout):
    """Once one wait gave up, later waits on the device give up at their first poll (one dead
    peer ends every wait within one poll, not one timeout each) until the host clears it."""
    from paper_2411_18889_b200 import _lib

    lib = _lib.load()
    ny, nz = 4, 8
    f = torch.rand((4, ny, nz), device="cuda")
    fn = torch.empty_like(f)
    mbox = torch.zeros(int(lib.b2_diffusion3d_mailbox_bytes(ny, nz)), dtype=torch.uint8, device="cuda")
    edges = lambda: lib.b2_diffusion3d_slab_edges(4, ny, nz, 0.1, 0.1, 0.1, 1e-3, 1.0, f.data_ptr(),  # noqa: E731
                                                  fn.data_ptr(), mbox.data_ptr(), None, None, None, 0, 0,
                                                  _lib.stream_handle())
    edges()
    torch.cuda.synchronize()
    lib.b2_set_poll_timeout_ms(60_000)  # a fresh wait would now take a minute...
    t0 = time.time()
    edges()
    torch.cuda.synchronize()
    assert time.time() - t0 < 5  # ...but the standing fault ends it at once
    with pytest.raises(_lib.SolomonError):
        _lib.check_fault()


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _stalled_peer_worker(rank, world, port, out):
    """Rank 1 stalls on the host far past the poll timeout before stepping: every rank's
    SlabDiffusion.synchronize raises SolomonError (no hang, no trap), and afterwards the
    process still computes on the GPU."""
    import torch.distributed as dist

    from paper_2411_18889_b200 import _lib
    from paper_2411_18889_b200.distributed import SlabDiffusion

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    _lib.set_poll_timeout(0.5)
    f0 = torch.rand((4, 8, 32), device="cuda", generator=torch.Generator("cuda").manual_seed(rank))
    sim = SlabDiffusion(f0, 0.1, 0.1, 0.1, 1e-3, 1.0, transport="p2p")
    if rank == 1:
        time.sleep(2.0)
    t0 = time.time()
    sim.step(3)
    err = None
    try:
        sim.synchronize()
    except _lib.SolomonError as e:
        err = str(e)
    waited = time.time() - t0
    x = torch.arange(1000, device="cuda", dtype=torch.float32).sum().item()  # the context survived
    res = [None] * world
    dist.all_gather_object(res, (err, waited, x))
    sim._closed = True  # the exchange is broken; just unmap
    if rank == 0:
        np.save(out, np.array(res, dtype=object), allow_pickle=True)
    dist.destroy_process_group()


def test_stalled_peer_fails_every_rank_cleanly(tmp_path):
    import torch.multiprocessing as mp

    out = tmp_path / "stall.npy"
    mp.spawn(_stalled_peer_worker, args=(2, _port(), str(out)), nprocs=2, join=True)
    res = np.load(out, allow_pickle=True)
    for err, waited, x in res:
        assert x == 499500.0
        assert waited < 30
    assert res[0][0] is not None and "timed out" in res[0][0]  # rank 0 waited for rank 1 and gave up
