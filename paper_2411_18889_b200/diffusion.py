"""7-point 3D diffusion on B200: the diffusion3d step, a device-resident time loop, grid setup.

``diffusion3d`` keeps the exact name, argument order and meaning of
``pkg/tests/fixtures/listing_diffusion.c:5``
(``diffusion3d(nx, ny, nz, dx, dy, dz, dt, kappa, f, fn)``) with CUDA
tensors as ``f`` / ``fn``; it runs the sm_100a marching kernel in
``csrc/diffusion.cu``. The buffers follow the reference's
``INDEX = k + nz*(j + ny*i)`` (listing_diffusion.c:1): a C-contiguous
``float32[nx, ny, nz]`` tensor. Like ``ACC_CLAUSE_PRESENT(f, fn)``
(listing_diffusion.c:10) the data must already be device-resident.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import torch

from ._lib import check, check_fault, load, on_device, require_cuda, stream_handle

_planned: set[tuple] = set()  # (shape, device, nsteps class) already passed to b2_diffusion3d_plan


def plan(f: torch.Tensor, fn: torch.Tensor, dx: float, dy: float, dz: float, dt: float, kappa: float,
         nsteps: int = 1) -> None:
    """Set-up call (b2_diffusion3d_plan): time the tile plans of this grid shape on ``f`` (read)
    and ``fn`` (written: scratch) and, for ``nsteps >= 2``, of the multi-step kernels, and size
    the resident path's mailbox. Host-synchronising, once per shape and device; the step and
    run calls then stay stream-ordered. Plans change time, never bits."""
    nx, ny, nz = f.shape
    key = (nx, ny, nz, f.device, min(int(nsteps), 2))
    if key in _planned:
        return
    with on_device(f.device):
        check(load().b2_diffusion3d_plan(nx, ny, nz, dx, dy, dz, dt, kappa, f.data_ptr(), fn.data_ptr(), int(nsteps),
                                         stream_handle(f.device)), "diffusion3d_plan")
    _planned.add(key)


def _grid(t: torch.Tensor, n: int, name: str) -> None:
    require_cuda(t, name)
    if t.dtype != torch.float32:
        raise TypeError(f"{name} must be float32 (listing_diffusion.c:5), got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous (INDEX = k + nz*(j + ny*i))")
    if t.numel() < n:
        raise ValueError(f"{name} has {t.numel()} cells, need {n}")


def coefficients(dx: float, dy: float, dz: float, dt: float, kappa: float) -> dict[str, float]:
    """ce, cn, ct, cc as listing_diffusion.c:6-9 (stable iff cc >= 0)."""
    import numpy as np

    f = np.float32
    kd = f(kappa) * f(dt)
    ce, cn, ct = kd / (f(dx) * f(dx)), kd / (f(dy) * f(dy)), kd / (f(dz) * f(dz))
    cc = f(1.0) - (((((ce + ce) + cn) + cn) + ct) + ct)
    return {"cc": float(cc), "ce": float(ce), "cw": float(ce), "cn": float(cn), "cs": float(cn),
            "ct": float(ct), "cb": float(ct)}


def diffusion3d(nx: int, ny: int, nz: int, dx: float, dy: float, dz: float, dt: float, kappa: float,
                f: torch.Tensor, fn: torch.Tensor) -> None:
    """One explicit step ``fn = f + kappa dt lap(f)`` with clamped boundaries (listing_diffusion.c:5-25).

    Stream-ordered on the current CUDA stream; bit-identical to the reference's -O3 build.
    The first call for a grid shape on a device plans its tiles (``plan``: host-synchronising
    once, before the step, writing ``fn``).
    """
    n = nx * ny * nz
    _grid(f, n, "f")
    _grid(fn, n, "fn")
    if f.data_ptr() == fn.data_ptr():
        raise ValueError("f and fn must not alias (restrict, listing_diffusion.c:5)")
    if (nx, ny, nz, f.device, 1) not in _planned and not torch.cuda.is_current_stream_capturing():
        plan(f.view(nx, ny, nz) if f.numel() == n else f.flatten()[:n].view(nx, ny, nz),
             fn.view(nx, ny, nz) if fn.numel() == n else fn.flatten()[:n].view(nx, ny, nz), dx, dy, dz, dt, kappa, 1)
    with on_device(f.device):
        check(load().b2_diffusion3d(nx, ny, nz, dx, dy, dz, dt, kappa, f.data_ptr(), fn.data_ptr(),
                                    stream_handle(f.device)), "diffusion3d")


def diffusion3d_slab(f: torch.Tensor, fn: torch.Tensor, halo_lo: torch.Tensor | None, halo_hi: torch.Tensor | None,
                     dx: float, dy: float, dz: float, dt: float, kappa: float, i_begin: int = 0,
                     i_end: int | None = None) -> None:
    """Slab step for i-decomposed grids (b2_diffusion3d_slab): ``f`` is ``[nx_local, ny, nz]``;
    ``halo_lo``/``halo_hi`` are the neighbours' edge planes or None at a global boundary."""
    nx, ny, nz = f.shape
    _grid(f, f.numel(), "f")
    _grid(fn, f.numel(), "fn")
    for h, name in ((halo_lo, "halo_lo"), (halo_hi, "halo_hi")):
        if h is not None:
            _grid(h, ny * nz, name)
    ptr = lambda t: t.data_ptr() if t is not None else None  # noqa: E731
    i_end = nx if i_end is None else i_end
    with on_device(f.device):
        check(load().b2_diffusion3d_slab(nx, ny, nz, dx, dy, dz, dt, kappa, f.data_ptr(), ptr(halo_lo),
                                         ptr(halo_hi), fn.data_ptr(), i_begin, i_end, stream_handle(f.device)),
              "diffusion3d_slab")


@dataclass
class Diffusion3D:
    """Device-resident time loop with ping-pong buffers.

    ``run(n)`` advances ``n`` steps with no host synchronisation; ``field``
    is the current solution.
    """

    f: torch.Tensor
    dx: float
    dy: float
    dz: float
    dt: float
    kappa: float = 1.0
    _fn: torch.Tensor = field(init=False, repr=False)

    def __post_init__(self) -> None:
        if self.f.dim() != 3:
            raise ValueError("f must be [nx, ny, nz]")
        _grid(self.f, self.f.numel(), "f")
        self._fn = torch.empty_like(self.f)
        self.steps = 0
        if not torch.cuda.is_current_stream_capturing():
            plan(self.f, self._fn, self.dx, self.dy, self.dz, self.dt, self.kappa, nsteps=2)

    def synchronize(self) -> None:
        """Wait for the queued steps; raises SolomonError if a device-side wait gave up
        (the resident path's bricks exchange faces in the GPU; b2_fault_status)."""
        check_fault(self.f.device, "Diffusion3D.run")

    @property
    def field(self) -> torch.Tensor:
        return self.f

    def run(self, nsteps: int) -> torch.Tensor:
        """Advance ``nsteps`` (b2_diffusion3d_run: two steps per HBM pass on large grids)."""
        nx, ny, nz = self.f.shape
        in_fn = ctypes.c_int(0)
        with on_device(self.f.device):
            check(load().b2_diffusion3d_run(nx, ny, nz, self.dx, self.dy, self.dz, self.dt, self.kappa,
                                            self.f.data_ptr(), self._fn.data_ptr(), int(nsteps), ctypes.byref(in_fn),
                                            stream_handle(self.f.device)), "diffusion3d_run")
        if in_fn.value:
            self.f, self._fn = self._fn, self.f
        self.steps += int(nsteps)
        return self.f

    # ---- checkpoint / resume -----------------------------------
    def state_dict(self) -> dict:
        return {"kind": "Diffusion3D", "f": self.f.clone(), "dx": self.dx, "dy": self.dy, "dz": self.dz,
                "dt": self.dt, "kappa": self.kappa, "steps": self.steps}

    def load_state_dict(self, sd: dict) -> None:
        if sd.get("kind") != "Diffusion3D":
            raise ValueError(f"not a Diffusion3D checkpoint: {sd.get('kind')!r}")
        if tuple(sd["f"].shape) != tuple(self.f.shape):
            raise ValueError(f"checkpoint grid {tuple(sd['f'].shape)} != {tuple(self.f.shape)}")
        if (sd["dx"], sd["dy"], sd["dz"], sd["dt"], sd["kappa"]) != (self.dx, self.dy, self.dz, self.dt, self.kappa):
            raise ValueError("checkpoint coefficients differ from this run's")
        self.f.copy_(sd["f"])
        self.steps = int(sd["steps"])

    @classmethod
    def from_state_dict(cls, sd: dict, device: torch.device | str = "cuda") -> "Diffusion3D":
        sim = cls(sd["f"].to(device).clone(), sd["dx"], sd["dy"], sd["dz"], sd["dt"], sd["kappa"])
        sim.steps = int(sd["steps"])
        return sim


def init_grid(nx: int, ny: int, nz: int, kind: str = "uniform", seed: int = 7,
              device: torch.device | str = "cuda") -> torch.Tensor:
    """Synthetic initial field: U[0,1) (seeded) or a Gaussian blob.

    Setup, not the hot path: generated with torch on ``device``.
    """
    if kind == "uniform":
        g = torch.Generator(device=device).manual_seed(seed)
        return torch.rand((nx, ny, nz), generator=g, dtype=torch.float32, device=device)
    if kind == "blob":
        axes = [(torch.arange(n, device=device, dtype=torch.float32) + 0.5) / n - 0.5 for n in (nx, ny, nz)]
        x, y, z = torch.meshgrid(*axes, indexing="ij")
        return torch.exp(-(x * x + y * y + z * z) / (2 * 0.05 ** 2)).contiguous()
    raise ValueError(f"unknown grid kind {kind!r}")
