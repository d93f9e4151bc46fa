"""Partitioning across one 8xB200 box.

One process per GPU, ``torch.distributed`` (NCCL over NVLink/NVSwitch) for
the plumbing. The reference is single-device; both
strategies here are new and keep the reference's per-element arithmetic, so
a sharded run is bit-identical to the unsharded one:

* N-body -- i-particle shards. Each rank owns a contiguous block of N/P
  particles (pos, vel, acc). Per step: all-gather positions (16 B/particle,
  in place into the shared ``pos_all`` buffer), force of local i against all
  j (listing_nbody.c:1 already separates the i set from the j set), fused
  local KDK update. j-chunking depends on N only, so summation order matches
  P = 1.
* Diffusion -- slabs along i, the slowest axis of INDEX (listing_diffusion.c:1;
  BASELINE's "z-slab"). Per step: exchange one ny*nz plane with each
  neighbour (grouped NCCL send/recv on a comm stream) while the interior
  planes compute, then the two boundary planes. Global ends clamp exactly as
  IMAX(i-1,0) / IMIN(i+1,nx-1).

The compute backend is injectable (``kernels=``) only so the exchange logic
can be tested on CPU with gloo; the default is the sm_100a library and it
fails loudly without it.
"""
from __future__ import annotations

import ctypes
import datetime
import os
from dataclasses import dataclass

import torch
import torch.distributed as dist

from . import _lib
from ._lib import B2_KDK_KICK_DRIFT, B2_KDK_KICK_END, B2_KDK_REDUCE


# ---------------------------------------------------------------------------
# Compute backends

class CudaNBodyKernels:
    """The sm_100a kernels (csrc/nbody.cu) via the C-ABI."""

    def __init__(self, potential: bool = False, exact: bool = False):
        self.flags = (_lib.B2_POTENTIAL if potential else 0) | (_lib.B2_EXACT if exact else 0)
        self.lib = _lib.load()

    def nchunks(self, nj: int) -> int:
        return self.lib.b2_calc_acc_nchunks(nj, self.flags)

    def workspace_bytes(self, ni: int, nj: int) -> int:
        return int(self.lib.b2_calc_acc_workspace_bytes(ni, nj, self.flags))

    def force(self, ipos: torch.Tensor, jpos: torch.Tensor, eps: float, acc: torch.Tensor, ws: torch.Tensor) -> None:
        """acc = calc_acc(ipos, jpos) with the chunk partials reduced in order inside the kernel
        (b2_calc_acc; the same bits as partials + B2_KDK_REDUCE)."""
        _lib.check(self.lib.b2_calc_acc(ipos.shape[0], ipos.data_ptr(), acc.data_ptr(), jpos.shape[0],
                                        jpos.data_ptr(), float(eps), self.flags, ws.data_ptr(), ws.numel(),
                                        _lib.stream_handle(ipos.device)), "calc_acc")

    def partials(self, ipos: torch.Tensor, jpos: torch.Tensor, eps: float, out: torch.Tensor) -> None:
        _lib.check(self.lib.b2_calc_acc_partials(ipos.shape[0], ipos.data_ptr(), jpos.shape[0], jpos.data_ptr(),
                                                 float(eps), self.flags, out.data_ptr(),
                                                 _lib.stream_handle(ipos.device)), "calc_acc_partials")

    def update(self, pos, vel, acc, partials, nchunks, h_end, h_begin, dt, phases) -> None:
        ptr = lambda t: t.data_ptr() if t is not None else None  # noqa: E731
        _lib.check(self.lib.b2_kdk_update(acc.shape[0], ptr(pos), ptr(vel), acc.data_ptr(), ptr(partials), nchunks,
                                          float(h_end), float(h_begin), float(dt), phases,
                                          _lib.stream_handle(acc.device)), "kdk_update")


class CudaSlabKernels:
    def __init__(self, dx, dy, dz, dt, kappa):
        self.args = (dx, dy, dz, dt, kappa)
        self.lib = _lib.load()

    def slab(self, f, fn, halo_lo, halo_hi, i_begin, i_end) -> None:
        """Halo arguments are tensors, raw device addresses (peer memory) or None."""
        nx, ny, nz = f.shape
        ptr = lambda t: t if (t is None or isinstance(t, int)) else t.data_ptr()  # noqa: E731
        _lib.check(self.lib.b2_diffusion3d_slab(nx, ny, nz, *self.args, f.data_ptr(), ptr(halo_lo), ptr(halo_hi),
                                                fn.data_ptr(), i_begin, i_end, _lib.stream_handle(f.device)),
                   "diffusion3d_slab")


    def plan(self, f, fn, nsteps) -> None:
        """Tile plans for this slab shape (b2_diffusion3d_plan; set-up, host-synchronising)."""
        from .diffusion import plan

        plan(f, fn, *self.args, nsteps=nsteps)

    def run2(self, f, fn) -> bool:
        """Two steps over a (halo-extended) slab; True when the result is in fn."""
        nx, ny, nz = f.shape
        in_fn = ctypes.c_int(0)
        _lib.check(self.lib.b2_diffusion3d_run(nx, ny, nz, *self.args, f.data_ptr(), fn.data_ptr(), 2,
                                               ctypes.byref(in_fn), _lib.stream_handle(f.device)), "diffusion3d_run")
        return bool(in_fn.value)

    def run2_planes(self, f, fn, p0: int, p1: int, p2: int = 0, p3: int = 0) -> bool:
        """Two steps over a (halo-extended) slab written only to fn[p0:p1] and fn[p2:p3]
        (b2_diffusion3d_run2_planes); False when the shape has no kernel for it."""
        nx, ny, nz = f.shape
        rc = self.lib.b2_diffusion3d_run2_planes(nx, ny, nz, *self.args, f.data_ptr(), fn.data_ptr(), p0, p1, p2, p3,
                                                  _lib.stream_handle(f.device))
        if rc == _lib.B2_ENOTSUP:
            return False
        _lib.check(rc, "diffusion3d_run2_planes")
        return True


def _all_gather_inplace(out: torch.Tensor, local: torch.Tensor, group=None) -> None:
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(out, local, group=group)
        return
    world = dist.get_world_size(group)
    parts = list(out.chunk(world))
    dist.all_gather(parts, local.clone(), group=group)


class _CudaArray:
    """__cuda_array_interface__ of raw device memory, for a zero-copy torch view."""

    def __init__(self, ptr: int, shape: tuple, typestr: str = "<f4"):
        self.__cuda_array_interface__ = {"shape": shape, "typestr": typestr, "data": (ptr, False), "version": 3,
                                         "strides": None}


def _device_view(ptr: int, shape: tuple, device: torch.device) -> torch.Tensor:
    return torch.as_tensor(_CudaArray(ptr, shape), device=device)


def init_distributed(backend: str = "nccl", timeout_s: float = 600.0) -> tuple[int, int, int]:
    """One process per GPU (torchrun env: RANK, WORLD_SIZE, LOCAL_RANK, MASTER_*).

    Binds the process to its GPU, defaults the rendezvous to 127.0.0.1, and sets a
    collective timeout so a lost peer fails the job instead of hanging it (SURVEY.md
    §5: failure detection = NCCL timeouts; nothing elastic). Returns (rank, world,
    local_rank).
    """
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29511")
    kw = {}
    if backend == "nccl":
        torch.cuda.set_device(local)
        kw["device_id"] = torch.device("cuda", local)
    dist.init_process_group(backend, rank=rank, world_size=world, timeout=datetime.timedelta(seconds=timeout_s),
                            **kw)
    return rank, world, local


# ---------------------------------------------------------------------------
# N-body

@dataclass
class ShardPlan:
    n_total: int
    world: int
    rank: int

    @property
    def n_local(self) -> int:
        return self.n_total // self.world

    @property
    def lo(self) -> int:
        return self.rank * self.n_local

    @property
    def hi(self) -> int:
        return self.lo + self.n_local


def shard_plan(n_total: int, group=None) -> ShardPlan:
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    if n_total % world:
        raise ValueError(f"N={n_total} must be divisible by the world size {world}")
    return ShardPlan(n_total, world, rank)


class ShardedLeapfrog:
    """KDK leapfrog with i-particle shards.

    ``pos_local``/``vel_local`` are this rank's block (rows [lo, hi) of the
    global arrays). ``pos_all`` holds every rank's positions.

    ``transport="nccl"``: positions are all-gathered in place with NCCL before
    every force evaluation.

    ``transport="p2p"`` (fused all-gather): ``pos_all`` is double-buffered and
    every rank maps every peer's two buffers (CUDA IPC). The update kernel that
    drifts the positions stores them into all peers' next buffer as it writes
    its own (``b2_kdk_update_publish``) -- the all-gather happens inside the
    producing kernel. Before a force evaluation each rank's stream waits on all
    peers' post-update interprocess events (a CPU-only gloo barrier makes sure
    they were recorded). Double buffering removes the write-after-read hazard:
    update k writes the buffer last read by force k-1, and every peer's force k
    waits on all updates k-1, each of which followed that peer's force k-1.

    ``transport="nvls"`` (NVSwitch multicast): the two buffers are every rank's copy of one
    multicast object (``b2_mc_*``); the update kernel stores each new position ONCE through
    the multicast view (``b2_kdk_update_multicast``) and the switch writes it into all ranks'
    copies -- one store per particle instead of one per peer. Ordering as for ``p2p``.
    """

    _closed = False  # set by close(): stepping afterwards raises

    def __init__(self, pos_local: torch.Tensor, vel_local: torch.Tensor, eps: float, dt: float, *, group=None,
                 kernels=None, potential: bool = False, exact: bool = False, transport: str = "nccl"):
        if transport not in ("nccl", "p2p", "nvls"):
            raise ValueError(f"unknown transport {transport!r}")
        self.group = group
        self.transport = transport
        n_local = pos_local.shape[0]
        self.plan = shard_plan(n_local * dist.get_world_size(group), group)
        self.k = kernels or CudaNBodyKernels(potential, exact)
        dev = pos_local.device
        if transport == "nvls":
            self._bufs = self._setup_nvls(dev)  # the two buffers: this rank's copy of the multicast memory
        else:
            nbuf = 2 if transport == "p2p" else 1
            self._bufs = [torch.empty((self.plan.n_total, 4), dtype=torch.float32, device=dev) for _ in range(nbuf)]
        self._cur = 0
        self.pos.copy_(pos_local)
        self.vel = vel_local.clone()
        self.acc = torch.empty_like(self.pos)
        self.eps, self.dt = float(eps), float(dt)
        self.nch = self.k.nchunks(self.plan.n_total)
        # CUDA kernels: the force kernel reduces the chunk partials itself (L2 ring workspace);
        # injected test kernels: partials [nch][n_local] + the update's in-order reduce
        self.fused = hasattr(self.k, "force")
        if self.fused:
            self.ws = torch.empty(max(self.k.workspace_bytes(n_local, self.plan.n_total), 16), dtype=torch.uint8,
                                  device=dev)
            self.part = None
        else:
            self.part = torch.empty((max(self.nch, 1) * n_local, 4), dtype=torch.float32, device=dev)
        self._opened = False
        self.steps = 0
        if transport == "p2p":
            self._setup_p2p()
        elif transport == "nvls":
            self._setup_events()
        self.gather()
        self._force()
        if not self.fused:
            self.k.update(None, None, self.acc, self.part, self.nch, 0.0, 0.0, 0.0, B2_KDK_REDUCE)

    def _force(self) -> None:
        """This shard's accelerations from pos_all (fused: into acc; else: partials)."""
        if self.fused:
            self.k.force(self.pos, self.pos_all, self.eps, self.acc, self.ws)
        else:
            self.k.partials(self.pos, self.pos_all, self.eps, self.part)

    @property
    def reduce_phase(self) -> int:
        """B2_KDK_REDUCE when the update must reduce partials (unfused kernels), else 0."""
        return 0 if self.fused else B2_KDK_REDUCE

    @property
    def pos_all(self) -> torch.Tensor:
        return self._bufs[self._cur]

    @property
    def pos(self) -> torch.Tensor:
        return self._bufs[self._cur][self.plan.lo:self.plan.hi]  # contiguous view: in-place gather source

    # ---- p2p transport -------------------------------------------------------
    def _setup_p2p(self) -> None:
        lib = _lib.load()
        if not self.pos_all.is_cuda:
            raise ValueError("transport='p2p' needs CUDA tensors")
        self.ctrl = dist.new_group(backend="gloo") if dist.get_backend(self.group) != "gloo" else self.group
        world, rank = self.plan.world, self.plan.rank
        if world - 1 > 8:
            raise ValueError("p2p transport supports up to 9 ranks (8 peers per kernel)")
        hb = lib.b2_ipc_handle_bytes()
        mine = []
        for t in self._bufs:
            h = ctypes.create_string_buffer(hb)
            off = ctypes.c_size_t(0)
            _lib.check(lib.b2_ipc_export(t.data_ptr(), h, ctypes.byref(off)), "ipc_export")
            mine.append((h.raw, off.value))
        self.event = torch.cuda.Event(enable_timing=False, interprocess=True)
        self.event.record(torch.cuda.current_stream(self.pos_all.device))
        everyone = [None] * world
        dist.all_gather_object(everyone, {"bufs": mine, "event": bytes(self.event.ipc_handle())}, group=self.ctrl)
        self._peers = []  # (ptrs per buffer, opened handles, event)
        err = None
        try:
            for r in range(world):
                if r == rank:
                    continue
                ptrs, opened = [], []
                for h, off in everyone[r]["bufs"]:
                    p = ctypes.c_void_p()
                    _lib.check(lib.b2_ipc_import(ctypes.create_string_buffer(h, len(h)), off, ctypes.byref(p)),
                               "ipc_import")
                    ptrs.append(p.value)
                    opened.append((p.value, off))
                ev = torch.cuda.Event.from_ipc_handle(self.pos_all.device, everyone[r]["event"])
                self._peers.append((ptrs, opened, ev))
        except Exception as e:  # noqa: BLE001 -- agreed on below so that no rank is left in a collective
            err = e
        ok = torch.tensor([0 if err else 1], dtype=torch.int32)
        dist.all_reduce(ok, op=dist.ReduceOp.MIN, group=self.ctrl)
        if not int(ok.item()):
            self.close()
            raise _lib.SolomonError(f"p2p position transport unavailable on some rank: {err or 'peer failure'}")

    # ---- nvls transport (NVSwitch multicast) -----------------------------------
    def _agree(self, err, what: str) -> None:
        ok = torch.tensor([0 if err else 1], dtype=torch.int32)
        dist.all_reduce(ok, op=dist.ReduceOp.MIN, group=self.ctrl)
        if not int(ok.item()):
            raise _lib.SolomonError(f"{what} unavailable on some rank: {err or 'peer failure'}")

    def _setup_nvls(self, dev: torch.device) -> list:
        """Both position buffers in ONE multicast object (b2_mc_*): rank 0 creates it, every
        rank adds its GPU, then binds its own copy and maps the multicast view. The update
        kernel stores each new position once through the multicast view
        (b2_kdk_update_multicast) and the switch writes it into every rank's copy -- the NVLS
        all-gather. Events and the host barrier order the steps as for p2p."""
        lib = _lib.load()
        if dev.type != "cuda":
            raise ValueError("transport='nvls' needs CUDA tensors")
        self.ctrl = dist.new_group(backend="gloo") if dist.get_backend(self.group) != "gloo" else self.group
        world, rank = self.plan.world, self.plan.rank
        err = None if lib.b2_mc_supported(dev.index) else "no multicast (NVLS) support on this GPU"
        self._agree(err, "nvls transport")
        need = 2 * self.plan.n_total * 16
        size = ctypes.c_size_t(0)
        _lib.check(lib.b2_mc_granular_bytes(need, world, ctypes.byref(size)), "mc_granular_bytes")
        binding, handle, err = ctypes.c_void_p(), ctypes.create_string_buffer(lib.b2_mc_handle_bytes()), None
        if rank == 0:
            rc = lib.b2_mc_create(size.value, world, dev.index, handle, ctypes.byref(binding))
            err = None if rc == 0 else f"b2_mc_create: {lib.b2_error_string(rc).decode()} ({rc})"
        shared = [handle.raw if rank == 0 else None]
        dist.broadcast_object_list(shared, src=dist.get_global_rank(self.ctrl, 0) if self.ctrl is not None else 0,
                                   group=self.ctrl)
        if rank != 0 and shared[0] is not None:
            h = ctypes.create_string_buffer(shared[0], len(shared[0]))
            rc = lib.b2_mc_add_device(h, dev.index, ctypes.byref(binding))
            err = None if rc == 0 else f"b2_mc_add_device: {lib.b2_error_string(rc).decode()} ({rc})"
        try:
            self._agree(err, "nvls transport")  # every GPU added before anyone binds
        except _lib.SolomonError:
            if binding.value:
                lib.b2_mc_release(binding)
            raise
        uc, mc = ctypes.c_void_p(), ctypes.c_void_p()
        rc = lib.b2_mc_bind(binding, size.value, ctypes.byref(uc), ctypes.byref(mc))
        err = None if rc == 0 else f"b2_mc_bind: {lib.b2_error_string(rc).decode()} ({rc})"
        try:
            self._agree(err, "nvls transport")
        except _lib.SolomonError:
            lib.b2_mc_release(binding)
            raise
        self._mc = (binding, uc.value, mc.value)
        n = self.plan.n_total
        return [_device_view(uc.value + b * n * 16, (n, 4), dev) for b in range(2)]

    def _setup_events(self) -> None:
        """The peers' post-update interprocess events (nvls; p2p sets them up with its mappings)."""
        self.event = torch.cuda.Event(enable_timing=False, interprocess=True)
        self.event.record(torch.cuda.current_stream(self.pos_all.device))
        everyone = [None] * self.plan.world
        dist.all_gather_object(everyone, bytes(self.event.ipc_handle()), group=self.ctrl)
        self._peers = [([], [], torch.cuda.Event.from_ipc_handle(self.pos_all.device, h))
                       for r, h in enumerate(everyone) if r != self.plan.rank]

    def _mc_slice(self, buf: int) -> int:
        """Multicast address of this rank's slice of buffer ``buf``."""
        if self._closed:
            raise RuntimeError("ShardedLeapfrog: the nvls transport was closed")
        return self._mc[2] + (buf * self.plan.n_total + self.plan.lo) * 16

    def _peer_ptrs(self, buf: int):
        if self._closed:
            raise RuntimeError("ShardedLeapfrog: the p2p transport was closed")
        off = self.plan.lo * 16  # our slice inside each peer's buffer
        arr = (ctypes.c_void_p * max(len(self._peers), 1))(*[p[0][buf] + off for p in self._peers])
        return arr, len(self._peers)

    def _publish_update(self, vel, partials, h_end, h_begin, dt, phases) -> None:
        """Update + store the resulting positions into the next buffer here and on every peer."""
        nxt = 1 - self._cur
        ptr = lambda t: t.data_ptr() if t is not None else None  # noqa: E731
        if self.transport == "nvls":
            _lib.check(_lib.load().b2_kdk_update_multicast(
                self.acc.shape[0], self.pos.data_ptr(), self._mc_slice(nxt), ptr(vel), self.acc.data_ptr(),
                ptr(partials), self.nch, float(h_end), float(h_begin), float(dt), phases,
                _lib.stream_handle(self.acc.device)), "kdk_update_multicast")
        else:
            peers, npeers = self._peer_ptrs(nxt)
            dst = self._bufs[nxt][self.plan.lo:self.plan.hi]
            _lib.check(_lib.load().b2_kdk_update_publish(
                self.acc.shape[0], self.pos.data_ptr(), dst.data_ptr(), ptr(vel), self.acc.data_ptr(), ptr(partials),
                self.nch, float(h_end), float(h_begin), float(dt), phases, peers, npeers,
                _lib.stream_handle(self.acc.device)), "kdk_update_publish")
        self.event.record(torch.cuda.current_stream(self.acc.device))
        self._cur = nxt

    def _await_peers(self) -> None:
        dist.barrier(group=self.ctrl)  # host-side: every peer recorded its latest post-update event
        stream = torch.cuda.current_stream(self.pos_all.device)
        for _, _, ev in self._peers:
            stream.wait_event(ev)

    def close(self) -> None:
        if self.transport == "nccl" or self._closed:
            return
        self._closed = True
        torch.cuda.synchronize(self.pos_all.device)
        dist.barrier(group=self.ctrl)
        lib = _lib.load()
        for _, opened, _ in self._peers:
            for p, off in opened:
                lib.b2_ipc_close(p, off)
        self._peers = []
        if self.transport == "nvls":
            self._bufs = [b.clone() for b in self._bufs]  # keep the state readable after the unmap
            lib.b2_mc_release(self._mc[0])
            self._mc = None
        dist.barrier(group=self.ctrl)

    # ---- stepping --------------------------------------------------------------
    def gather(self) -> None:
        """Make pos_all hold every rank's current positions."""
        if self.transport == "nccl":
            _all_gather_inplace(self.pos_all, self.pos, self.group)
            return
        # publish our slice of the current buffer into every peer's current buffer
        if self.transport == "nvls":
            _lib.check(_lib.load().b2_kdk_update_multicast(
                self.pos.shape[0], self.pos.data_ptr(), self._mc_slice(self._cur), None, self.pos.data_ptr(), None,
                1, 0.0, 0.0, 0.0, 0, _lib.stream_handle(self.pos.device)), "publish")
        else:
            peers, npeers = self._peer_ptrs(self._cur)
            _lib.check(_lib.load().b2_kdk_update_publish(
                self.pos.shape[0], self.pos.data_ptr(), self.pos.data_ptr(), None, self.pos.data_ptr(), None, 1,
                0.0, 0.0, 0.0, 0, peers, npeers, _lib.stream_handle(self.pos.device)), "publish")
        self.event.record(torch.cuda.current_stream(self.pos.device))
        self._await_peers()

    def step(self, nsteps: int = 1, *, close: bool = True) -> None:
        """Advance ``nsteps``; with ``close`` the velocities are synchronised (closing half-kick applied)."""
        h = 0.5 * self.dt
        for s in range(nsteps):
            if self.transport == "nccl":
                if not self._opened:
                    self.k.update(self.pos, self.vel, self.acc, None, self.nch, 0.0, h, self.dt, B2_KDK_KICK_DRIFT)
                    self._opened = True
                self.gather()
                self._force()
                last = close and s + 1 == nsteps
                phases = self.reduce_phase | B2_KDK_KICK_END | (0 if last else B2_KDK_KICK_DRIFT)
                self.k.update(self.pos, self.vel, self.acc, self.part, self.nch, h, h, self.dt, phases)
                self._opened = not last
            else:
                if not self._opened:
                    # WAR: the buffer this update publishes into was read by the peers'
                    # last force evaluation -- wait for their last update (which followed it).
                    self._await_peers()
                    self._publish_update(self.vel, None, 0.0, h, self.dt, B2_KDK_KICK_DRIFT)
                    self._opened = True
                self._await_peers()
                self._force()
                last = close and s + 1 == nsteps
                phases = self.reduce_phase | B2_KDK_KICK_END | (0 if last else B2_KDK_KICK_DRIFT)
                self._publish_update(self.vel, self.part, h, h, self.dt, phases)
                self._opened = not last
            self.steps += 1

    def launches_per_step(self) -> int:
        return 2

    def synchronize(self) -> None:
        """Wait for this rank's queued steps; raises SolomonError if a device-side wait gave up."""
        if self.pos_all.is_cuda:
            _lib.check_fault(self.pos_all.device, "ShardedLeapfrog.step")

    # ---- checkpoint / resume -----------------------------------
    def state_dict(self) -> dict:
        """This rank's shard. ``opened`` records a pending opening half-kick
        (``step(close=False)``), so a resumed run continues bit for bit."""
        return {"kind": "ShardedLeapfrog", "n_total": self.plan.n_total, "world": self.plan.world,
                "rank": self.plan.rank, "pos": self.pos.clone(), "vel": self.vel.clone(), "acc": self.acc.clone(),
                "eps": self.eps, "dt": self.dt, "opened": self._opened, "steps": self.steps}

    def load_state_dict(self, sd: dict) -> None:
        """Collective: every rank loads its own shard, then positions are re-gathered."""
        if sd.get("kind") != "ShardedLeapfrog":
            raise ValueError(f"not a ShardedLeapfrog checkpoint: {sd.get('kind')!r}")
        want = (self.plan.n_total, self.plan.world, self.plan.rank)
        if (sd["n_total"], sd["world"], sd["rank"]) != want:
            raise ValueError(f"checkpoint is for (N, world, rank) = {(sd['n_total'], sd['world'], sd['rank'])}, "
                             f"this run is {want}")
        if (sd["eps"], sd["dt"]) != (self.eps, self.dt):
            raise ValueError("checkpoint eps/dt differ from this run's")
        self.pos.copy_(sd["pos"])
        self.vel.copy_(sd["vel"])
        self.acc.copy_(sd["acc"])
        self._opened = bool(sd["opened"])
        self.steps = int(sd["steps"])
        self.gather()


# ---------------------------------------------------------------------------
# Diffusion

class SlabDiffusion:
    """Explicit diffusion on i-slabs with a one-plane halo exchange per step.

    ``f_local`` is this rank's ``[nx_local, ny, nz]`` block of the global grid
    (planes [rank*nx_local, (rank+1)*nx_local) for equal splits; ranks may
    differ in nx_local).

    ``transport="nccl"``: the two edge planes go to the neighbours with grouped
    NCCL send/recv on a comm stream while the interior computes.

    ``transport="p2p"`` (fused halo, no collective, no host synchronisation per
    step): every rank maps its neighbours' halo mailboxes once (CUDA IPC; peer
    access over NVLink/NVSwitch). Each step is the interior-plane launch plus one
    edge-plane kernel (b2_diffusion3d_slab_edges) that polls its own mailbox for
    the neighbours' rows of the current state -- self-validating 16-byte words
    {value, tag, value, tag} -- computes the two edge planes and stores its new edge
    rows straight into the neighbours' mailboxes.
    """

    _closed = False  # set by close(): stepping afterwards raises

    def __init__(self, f_local: torch.Tensor, dx, dy, dz, dt, kappa=1.0, *, group=None, kernels=None,
                 transport: str = "nccl"):
        if f_local.dim() != 3 or f_local.shape[0] < 2:
            raise ValueError("f_local must be [nx_local >= 2, ny, nz]")
        if transport not in ("nccl", "p2p"):
            raise ValueError(f"unknown transport {transport!r}")
        self.group = group
        self.world, self.rank = dist.get_world_size(group), dist.get_rank(group)
        self.k = kernels or CudaSlabKernels(dx, dy, dz, dt, kappa)
        nxl, ny, nz = f_local.shape
        self.has_lo = self.rank > 0
        self.has_hi = self.rank < self.world - 1
        # f / fn are views of two halo-extended slabs [2 halo | nx_local | 2 halo] (no halo at a
        # global end): step() works on the views, run() on the whole slabs without copies
        self._lo_h = 2 if self.has_lo else 0
        ext = (self._lo_h + nxl + (2 if self.has_hi else 0), ny, nz)
        self._ext = (torch.zeros(ext, dtype=f_local.dtype, device=f_local.device),
                     torch.zeros(ext, dtype=f_local.dtype, device=f_local.device))
        self.f, self.fn = (e[self._lo_h:self._lo_h + nxl] for e in self._ext)
        self.f.copy_(f_local)
        self._agree_planes(ny, nz)
        self.is_cuda = self.f.is_cuda
        self.transport = transport
        self.steps_done = 0
        if self.is_cuda and hasattr(self.k, "plan"):  # set-up: time the tile plans once (writes fn: scratch)
            self.k.plan(self.f, self.fn, 1)  # step(): the interior planes of the slab
            self.k.plan(*self._ext, 2)       # run(): two steps per pass over the halo-extended slab
        if transport == "nccl":
            self.halo_lo = torch.empty((ny, nz), dtype=self.f.dtype, device=self.f.device) if self.has_lo else None
            self.halo_hi = torch.empty((ny, nz), dtype=self.f.dtype, device=self.f.device) if self.has_hi else None
            self.comm = torch.cuda.Stream(device=self.f.device) if self.is_cuda else None
        else:
            if not self.is_cuda:
                raise ValueError("transport='p2p' needs CUDA tensors")
            self._setup_p2p()

    def _agree_planes(self, ny: int, nz: int) -> None:
        """Every rank must hold [*, ny, nz] planes (a halo is one plane). Checked collectively,
        so a mismatch raises on every rank instead of deadlocking the first exchange."""
        dev = self.f.device if dist.get_backend(self.group) == "nccl" else torch.device("cpu")
        t = torch.tensor([ny, nz, -ny, -nz], dtype=torch.int64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self.group)
        hy, hz, ly, lz = (int(v) for v in t.tolist())
        if (hy, hz, -ly, -lz) != (ny, nz, ny, nz):
            raise ValueError(f"ranks hold different planes: ny in [{-ly}, {hy}], nz in [{-lz}, {hz}]")

    # ---- p2p transport -------------------------------------------------------
    def _setup_p2p(self) -> None:
        """Map the neighbours' halo mailboxes (CUDA IPC) and publish the state-0 edge planes.

        Host synchronisation happens here only (and in close / load_state_dict): once every
        rank has zeroed its mailbox, steps run with no barrier, event or collective -- the
        edge kernel polls its mailbox for tagged rows and pushes its own rows to the
        neighbours (b2_diffusion3d_slab_edges)."""
        lib = _lib.load()
        self.ctrl = dist.new_group(backend="gloo") if dist.get_backend(self.group) != "gloo" else self.group
        ny, nz = self.f.shape[1:]
        self._side_bytes = int(lib.b2_diffusion3d_mailbox_bytes(ny, nz))
        self._side2 = int(lib.b2_diffusion3d_mailbox2_bytes(ny, nz))
        # [per-step: fed by rank-1 | by rank+1][run(): fed by rank-1 | by rank+1]
        self.mbox = torch.zeros(2 * self._side_bytes + 2 * self._side2, dtype=torch.uint8, device=self.f.device)
        hb = lib.b2_ipc_handle_bytes()
        h = ctypes.create_string_buffer(hb)
        off = ctypes.c_size_t(0)
        _lib.check(lib.b2_ipc_export(self.mbox.data_ptr(), h, ctypes.byref(off)), "ipc_export")
        everyone = [None] * self.world
        dist.all_gather_object(everyone, (h.raw, off.value), group=self.ctrl)
        self._peer = {}  # rank -> (mapped mailbox base, offset)
        err = None
        try:
            for r in (self.rank - 1, self.rank + 1):
                if 0 <= r < self.world:
                    ph, poff = everyone[r]
                    ptr = ctypes.c_void_p()
                    _lib.check(lib.b2_ipc_import(ctypes.create_string_buffer(ph, len(ph)), poff, ctypes.byref(ptr)),
                               "ipc_import")
                    self._peer[r] = (ptr.value, poff)
        except Exception as e:  # noqa: BLE001 -- agreed on below so that no rank is left in a collective
            err = e
        ok = torch.tensor([0 if err else 1], dtype=torch.int32)
        dist.all_reduce(ok, op=dist.ReduceOp.MIN, group=self.ctrl)
        if not int(ok.item()):
            for p, poff in self._peer.values():
                lib.b2_ipc_close(p, poff)
            self._peer = {}
            raise _lib.SolomonError(f"p2p halo transport unavailable on some rank: {err or 'peer failure'}")
        base = self.mbox.data_ptr()
        self._in_lo = base if self.has_lo else None
        self._in_hi = base + self._side_bytes if self.has_hi else None
        self._out_lo = self._peer[self.rank - 1][0] + self._side_bytes if self.has_lo else None  # its side fed by rank+1
        self._out_hi = self._peer[self.rank + 1][0] if self.has_hi else None              # its side fed by rank-1
        r2 = 2 * self._side_bytes  # run() mailboxes, same layout after the per-step pair
        self._in2 = (base + r2 if self.has_lo else None, base + r2 + self._side2 if self.has_hi else None)
        self._out2 = (self._peer[self.rank - 1][0] + r2 + self._side2 if self.has_lo else None,
                      self._peer[self.rank + 1][0] + r2 if self.has_hi else None)
        self._side = torch.cuda.Stream(device=self.f.device)  # the edge kernel of step()
        self._state_ready = torch.cuda.Event()  # main stream at the start of a step
        self._edges_done = torch.cuda.Event()
        self._publish_edges()

    def _edges(self, push_only: bool) -> None:
        if self._closed:
            raise RuntimeError("SlabDiffusion: the p2p transport was closed")
        nxl, ny, nz = self.f.shape
        _lib.check(_lib.load().b2_diffusion3d_slab_edges(
            nxl, ny, nz, *self.k.args, self.f.data_ptr(), self.fn.data_ptr(), self._in_lo, self._in_hi,
            self._out_lo, self._out_hi, self.steps_done, int(push_only), _lib.stream_handle(self.f.device)),
            "diffusion3d_slab_edges")

    def _publish_edges(self) -> None:
        """(Re)start the per-step exchange at state steps_done: every per-step mailbox zero, then
        every rank pushes. (run()'s mailboxes keep their monotonic exchange tags.)"""
        self.mbox[:2 * self._side_bytes].zero_()
        torch.cuda.synchronize(self.f.device)
        dist.barrier(group=self.ctrl)
        self._edges(push_only=True)

    def close(self) -> None:
        if self.transport != "p2p" or self._closed:
            return
        self._closed = True
        torch.cuda.synchronize(self.f.device)
        dist.barrier(group=self.ctrl)
        lib = _lib.load()
        for p, poff in self._peer.values():
            lib.b2_ipc_close(p, poff)
        self._peer = {}
        dist.barrier(group=self.ctrl)

    # ---- stepping --------------------------------------------------------------
    def _exchange_ops(self):
        ops = []
        g = self.group
        if self.has_lo:
            ops.append(dist.P2POp(dist.isend, self.f[0], self.rank - 1, g))
            ops.append(dist.P2POp(dist.irecv, self.halo_lo, self.rank - 1, g))
        if self.has_hi:
            ops.append(dist.P2POp(dist.isend, self.f[-1], self.rank + 1, g))
            ops.append(dist.P2POp(dist.irecv, self.halo_hi, self.rank + 1, g))
        return ops

    def _step_nccl(self) -> None:
        nxl = self.f.shape[0]
        ops = self._exchange_ops()
        reqs = []
        if ops:
            if self.is_cuda:
                self.comm.wait_stream(torch.cuda.current_stream(self.f.device))
                with torch.cuda.stream(self.comm):
                    reqs = dist.batch_isend_irecv(ops)
            else:
                reqs = dist.batch_isend_irecv(ops)
        # interior planes need no halo and overlap the exchange
        if nxl > 2:
            self.k.slab(self.f, self.fn, None, None, 1, nxl - 1)
        for r in reqs:
            r.wait()
        self.k.slab(self.f, self.fn, self.halo_lo, self.halo_hi, 0, 1)
        self.k.slab(self.f, self.fn, self.halo_lo, self.halo_hi, nxl - 1, nxl)

    def _step_p2p(self) -> None:
        nxl = self.f.shape[0]
        main = torch.cuda.current_stream(self.f.device)
        self._state_ready.record(main)  # everything queued so far (previous step, user copies into f)
        if nxl > 2:  # interior planes need no halo
            self.k.slab(self.f, self.fn, None, None, 1, nxl - 1)
        # edge planes + halo exchange, synchronised on the device, on a second stream so the
        # wait for the neighbours' rows overlaps the interior launch (queued first, so its
        # CTAs take the SMs first; the edge kernel's small CTAs run beside them). Planes 0 and
        # nxl-1 of fn are the edge kernel's, 1..nxl-2 the interior's: disjoint writes.
        self._side.wait_event(self._state_ready)
        with torch.cuda.stream(self._side):
            self._edges(push_only=False)
        self._edges_done.record(self._side)
        main.wait_event(self._edges_done)

    def step(self, nsteps: int = 1) -> torch.Tensor:
        for _ in range(nsteps):
            if self.transport == "p2p":
                self._step_p2p()
            else:
                self._step_nccl()
            self.f, self.fn = self.fn, self.f
            self.steps_done += 1
        return self.f

    # ---- two steps per exchange ------------------------------------------------
    def run(self, nsteps: int) -> torch.Tensor:
        """Advance ``nsteps`` with TWO steps per halo exchange (collective, bit-identical to
        ``step(nsteps)``). ``f``/``fn`` are views of halo-extended slabs with two neighbour
        planes per side; a pass is one ``b2_diffusion3d_run(..., 2)`` over a whole one (on large slabs
        the two-steps-per-HBM-pass kernel), the two planes next to the halo are exact after
        two steps and the two halo planes are refreshed between passes (NCCL send/recv, or
        over peer memory with ``b2_diffusion3d_slab_halo2`` for transport="p2p"). An odd
        remainder step runs through ``step(1)``."""
        if nsteps < 0:
            raise ValueError("nsteps must be >= 0")
        pairs = nsteps // 2
        if pairs:
            nxl, lo_h = self.f.shape[0], self._lo_h
            cur, oth = self._ext if self.f.data_ptr() == self._ext[0][lo_h].data_ptr() else self._ext[::-1]
            # overlap: the planes that need no halo computed while it travels (world > 1, slabs
            # of >= 6 planes, a kernel that writes a plane range); else refresh, then the pass
            overlap = (self.world > 1 and nxl >= 6 and hasattr(self.k, "run2_planes")
                       and self.k.run2_planes(cur, oth, 0, 0))
            for _ in range(pairs):
                if overlap:
                    self._pass_overlapped(cur, oth, lo_h, nxl)
                    cur, oth = oth, cur
                    continue
                self._halo2(cur, lo_h, nxl)
                if self.k.run2(cur, oth):
                    cur, oth = oth, cur
            self.f, self.fn = cur[lo_h:lo_h + nxl], oth[lo_h:lo_h + nxl]
            self.steps_done += 2 * pairs
            if self.transport == "p2p":
                self._publish_edges()  # the per-step halo restarts at the new state
        if nsteps % 2:
            self.step(1)
        return self.f

    def _pass_overlapped(self, cur: torch.Tensor, oth: torch.Tensor, lo_h: int, nxl: int) -> None:
        """One two-step pass cur -> oth with the halo exchange overlapped: the neighbours' two
        edge planes travel (NCCL on the comm stream, or the p2p push on the side stream) while
        the planes that need no halo -- all but the two next to each neighbour -- are computed;
        then the two planes next to each halo. Output plane p reads input planes p-2 .. p+2 only,
        so every plane gets the bits of the whole-slab pass."""
        lo_e = lo_h + (2 if self.has_lo else 0)          # first plane that needs no low halo
        hi_e = lo_h + nxl - (2 if self.has_hi else 0)    # one past the last that needs no high halo
        if self.transport == "p2p":
            if self._closed:
                raise RuntimeError("SlabDiffusion: the p2p transport was closed")
            nx_ext, ny, nz = cur.shape
            xchg = getattr(self, "_xchg", 0)
            lib, main = _lib.load(), torch.cuda.current_stream(cur.device)
            halo2 = lambda phase, stream: _lib.check(lib.b2_diffusion3d_slab_halo2(  # noqa: E731
                nx_ext, ny, nz, lo_h, nxl, cur.data_ptr(), *self._in2, *self._out2, xchg, phase,
                stream.cuda_stream), "diffusion3d_slab_halo2")
            self._side.wait_stream(main)   # cur's edge planes are final
            halo2(0, self._side)           # push them to the neighbours, beside the interior
            self.k.run2_planes(cur, oth, lo_e, hi_e)
            halo2(1, main)                 # the neighbours' planes into cur's halo
            self._xchg = xchg + 1
            main.wait_stream(self._side)   # the push read cur: done before a pass overwrites it
        else:
            ops, g = [], self.group
            if self.has_lo:
                ops.append(dist.P2POp(dist.isend, cur[lo_h:lo_h + 2], self.rank - 1, g))
                ops.append(dist.P2POp(dist.irecv, cur[0:2], self.rank - 1, g))
            if self.has_hi:
                ops.append(dist.P2POp(dist.isend, cur[lo_h + nxl - 2:lo_h + nxl], self.rank + 1, g))
                ops.append(dist.P2POp(dist.irecv, cur[lo_h + nxl:lo_h + nxl + 2], self.rank + 1, g))
            if self.is_cuda:
                self.comm.wait_stream(torch.cuda.current_stream(cur.device))
                with torch.cuda.stream(self.comm):
                    reqs = dist.batch_isend_irecv(ops)
            else:
                reqs = dist.batch_isend_irecv(ops)
            self.k.run2_planes(cur, oth, lo_e, hi_e)
            for r in reqs:
                r.wait()  # NCCL: the current stream waits for the exchange; gloo: the host does
        self.k.run2_planes(cur, oth, lo_h, lo_e, hi_e, lo_h + nxl)  # both edges, one launch

    def _halo2(self, cur: torch.Tensor, lo_h: int, nxl: int) -> None:
        """Fill cur's halo planes with the neighbours' two edge planes of the same state."""
        if self.transport == "p2p":
            if self._closed:
                raise RuntimeError("SlabDiffusion: the p2p transport was closed")
            nx_ext, ny, nz = cur.shape
            xchg = getattr(self, "_xchg", 0)
            lib, sh = _lib.load(), _lib.stream_handle(cur.device)
            for phase in (0, 1):  # push everything, then wait for the neighbours' planes
                _lib.check(lib.b2_diffusion3d_slab_halo2(nx_ext, ny, nz, lo_h, nxl, cur.data_ptr(), *self._in2,
                                                         *self._out2, xchg, phase, sh), "diffusion3d_slab_halo2")
            self._xchg = xchg + 1
            return
        ops, g = [], self.group
        if self.has_lo:
            ops.append(dist.P2POp(dist.isend, cur[lo_h:lo_h + 2], self.rank - 1, g))
            ops.append(dist.P2POp(dist.irecv, cur[0:2], self.rank - 1, g))
        if self.has_hi:
            ops.append(dist.P2POp(dist.isend, cur[lo_h + nxl - 2:lo_h + nxl], self.rank + 1, g))
            ops.append(dist.P2POp(dist.irecv, cur[lo_h + nxl:lo_h + nxl + 2], self.rank + 1, g))
        if ops:
            for r in dist.batch_isend_irecv(ops):
                r.wait()

    def launches_per_step(self) -> int:
        interior = 1 if self.f.shape[0] > 2 else 0
        return interior + (1 if self.transport == "p2p" else 2)

    def synchronize(self) -> None:
        """Wait for this rank's queued steps; raises SolomonError if a device-side wait for a
        neighbour's halo gave up (p2p transport: the peer is dead or stalled past the poll
        timeout, ``_lib.set_poll_timeout``). The context stays usable; the slab does not."""
        if self.is_cuda:
            _lib.check_fault(self.f.device, f"SlabDiffusion (rank {self.rank})")

    # ---- checkpoint / resume -----------------------------------
    def state_dict(self) -> dict:
        return {"kind": "SlabDiffusion", "world": self.world, "rank": self.rank, "f": self.f.clone(),
                "steps": self.steps_done}

    def load_state_dict(self, sd: dict) -> None:
        """Collective: every rank loads its own slab; the halo exchange restarts at the
        loaded state."""
        if sd.get("kind") != "SlabDiffusion":
            raise ValueError(f"not a SlabDiffusion checkpoint: {sd.get('kind')!r}")
        if (sd["world"], sd["rank"]) != (self.world, self.rank) or tuple(sd["f"].shape) != tuple(self.f.shape):
            raise ValueError("checkpoint is for a different decomposition")
        s = int(sd["steps"])
        self.f.copy_(sd["f"])
        self.steps_done = s
        if self.transport == "p2p":
            self._publish_edges()  # restart the halo exchange at the loaded state
        else:
            if self.is_cuda:
                torch.cuda.current_stream(self.f.device).synchronize()
            dist.barrier(group=self.group)
