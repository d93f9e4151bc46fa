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
        nx, ny, nz = f.shape
        ptr = lambda t: t.data_ptr() if t is not None else None  # noqa: E731
        _lib.check(self.lib.b2_diffusion3d_slab(nx, ny, nz, *self.args, f.data_ptr(), ptr(halo_lo), ptr(halo_hi),
                                                fn.data_ptr(), i_begin, i_end, _lib.stream_handle(f.device)),
                   "diffusion3d_slab")


def _all_gather_inplace(out: torch.Tensor, local: torch.Tensor, group=None) -> None:
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(out, local, group=group)
        return
    world = dist.get_world_size(group)
    parts = list(out.chunk(world))
    dist.all_gather(parts, local.clone(), group=group)


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
    """KDK leapfrog with i-particle shards and a position all-gather per step.

    ``pos_local``/``vel_local`` are this rank's block (rows [lo, hi) of the
    global arrays). ``pos_all`` holds every rank's positions after a gather.
    """

    def __init__(self, pos_local: torch.Tensor, vel_local: torch.Tensor, eps: float, dt: float, *, group=None,
                 kernels=None, potential: bool = False, exact: bool = False):
        self.group = group
        n_local = pos_local.shape[0]
        self.plan = shard_plan(n_local * dist.get_world_size(group), group)
        self.k = kernels or CudaNBodyKernels(potential, exact)
        dev = pos_local.device
        self.pos_all = torch.empty((self.plan.n_total, 4), dtype=torch.float32, device=dev)
        self.pos = self.pos_all[self.plan.lo:self.plan.hi]  # contiguous view: in-place gather source
        self.pos.copy_(pos_local)
        self.vel = vel_local.clone()
        self.acc = torch.empty_like(self.pos)
        self.eps, self.dt = float(eps), float(dt)
        self.nch = self.k.nchunks(self.plan.n_total)
        self.part = torch.empty((max(self.nch, 1) * n_local, 4), dtype=torch.float32, device=dev)
        self._opened = False
        self.gather()
        self.k.partials(self.pos, self.pos_all, self.eps, self.part)
        self.k.update(None, None, self.acc, self.part, self.nch, 0.0, 0.0, 0.0, B2_KDK_REDUCE)

    def gather(self) -> None:
        _all_gather_inplace(self.pos_all, self.pos, self.group)

    def step(self, nsteps: int = 1, *, close: bool = True) -> None:
        """Advance ``nsteps``; with ``close`` the velocities are synchronised (closing half-kick applied)."""
        h = 0.5 * self.dt
        for s in range(nsteps):
            if not self._opened:
                self.k.update(self.pos, self.vel, self.acc, None, self.nch, 0.0, h, self.dt, B2_KDK_KICK_DRIFT)
                self._opened = True
            self.gather()
            self.k.partials(self.pos, self.pos_all, self.eps, self.part)
            last = close and s + 1 == nsteps
            phases = B2_KDK_REDUCE | B2_KDK_KICK_END | (0 if last else B2_KDK_KICK_DRIFT)
            self.k.update(self.pos, self.vel, self.acc, self.part, self.nch, h, h, self.dt, phases)
            self._opened = not last

    def launches_per_step(self) -> int:
        return 2


# ---------------------------------------------------------------------------
# Diffusion

class SlabDiffusion:
    """Explicit diffusion on i-slabs with a one-plane halo exchange per step.

    ``f_local`` is this rank's ``[nx_local, ny, nz]`` block of the global grid
    (planes [rank*nx_local, (rank+1)*nx_local)).
    """

    def __init__(self, f_local: torch.Tensor, dx, dy, dz, dt, kappa=1.0, *, group=None, kernels=None):
        if f_local.dim() != 3 or f_local.shape[0] < 2:
            raise ValueError("f_local must be [nx_local >= 2, ny, nz]")
        self.group = group
        self.world, self.rank = dist.get_world_size(group), dist.get_rank(group)
        self.k = kernels or CudaSlabKernels(dx, dy, dz, dt, kappa)
        self.f = f_local.contiguous().clone()
        self.fn = torch.empty_like(self.f)
        ny, nz = self.f.shape[1:]
        self.has_lo = self.rank > 0
        self.has_hi = self.rank < self.world - 1
        self.halo_lo = torch.empty((ny, nz), dtype=self.f.dtype, device=self.f.device) if self.has_lo else None
        self.halo_hi = torch.empty((ny, nz), dtype=self.f.dtype, device=self.f.device) if self.has_hi else None
        self.is_cuda = self.f.is_cuda
        self.comm = torch.cuda.Stream(device=self.f.device) if self.is_cuda else None

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

    def step(self, nsteps: int = 1) -> torch.Tensor:
        nxl = self.f.shape[0]
        for _ in range(nsteps):
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
            self.f, self.fn = self.fn, self.f
        return self.f

    def launches_per_step(self) -> int:
        return 3 if self.f.shape[0] > 2 else 2
