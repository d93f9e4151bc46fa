"""Direct-summation N-body on B200: force (calc_acc), leapfrog KDK, initial conditions.

Python mirror of the reference's n-body path. ``calc_acc`` keeps the exact
name, argument order and meaning of ``pkg/tests/fixtures/listing_nbody.c:1``
(``calc_acc(Ni, ipos, iacc, Nj, jpos, eps)``) with CUDA tensors as the
buffers; it runs the sm_100a kernels in ``csrc/nbody.cu`` through the C-ABI
(``include/solomon_b200.h``). The integrator and initial-condition
generators have no reference counterpart and are specified
in DESIGN.md §2.3-2.4.

Layout (listing_nbody.c:1,4-6,9,25): particles are ``float32[N, 4]`` rows
``{x, y, z, m}``; accelerations ``{ax, ay, az, pot}`` where ``pot`` is
``sum_j m_j / sqrt(r2)`` when the potential is requested (the
``-DCALCULATE_POTENTIAL`` build, listing_nbody.c:21-23) and 0 otherwise.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import B2_EXACT, B2_POTENTIAL, check, load, on_device, require_cuda, stream_handle


def _flags(potential: bool, exact: bool) -> int:
    return (B2_POTENTIAL if potential else 0) | (B2_EXACT if exact else 0)


def _particles(t: torch.Tensor, n: int, name: str) -> None:
    require_cuda(t, name)
    if t.dtype != torch.float32:
        raise TypeError(f"{name} must be float32 (listing_nbody.c uses float4), got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous (AoS float4 rows)")
    if t.numel() < 4 * n:
        raise ValueError(f"{name} holds {t.numel() // 4} particles, need {n}")
    if t.data_ptr() % 16:
        raise ValueError(f"{name} must be 16-byte aligned (float4)")


def workspace(Ni: int, Nj: int, potential: bool = False, exact: bool = False,
              device: torch.device | str | None = None) -> torch.Tensor:
    """Scratch for the j-chunk partial sums (caller-owned; see b2_calc_acc_workspace_bytes)."""
    nbytes = load().b2_calc_acc_workspace_bytes(Ni, Nj, _flags(potential, exact))
    return torch.empty(max(int(nbytes), 16), dtype=torch.uint8, device=device or "cuda")


def calc_acc(Ni: int, ipos: torch.Tensor, iacc: torch.Tensor, Nj: int, jpos: torch.Tensor, eps: float,
             *, potential: bool = False, exact: bool = False, ws: torch.Tensor | None = None) -> None:
    """``iacc[:Ni] = sum_{j<Nj} m_j (r_j - r_i) / (|r_j - r_i|^2 + eps^2)^{3/2}`` (listing_nbody.c:1-27).

    Stream-ordered on the current CUDA stream. ``exact=True`` selects the
    bit-for-bit reference arithmetic (IEEE ``1/sqrt``, sequential j); the
    default fast path agrees to FP32 tolerance.
    """
    lib = load()
    _particles(ipos, Ni, "ipos")
    _particles(iacc, Ni, "iacc")
    _particles(jpos, Nj, "jpos")
    flags = _flags(potential, exact)
    need = lib.b2_calc_acc_workspace_bytes(Ni, Nj, flags)
    if need and (ws is None or ws.numel() < need):
        ws = torch.empty(need, dtype=torch.uint8, device=ipos.device)
    wptr = ws.data_ptr() if ws is not None else None
    wlen = ws.numel() if ws is not None else 0
    with on_device(ipos.device):
        check(lib.b2_calc_acc(Ni, ipos.data_ptr(), iacc.data_ptr(), Nj, jpos.data_ptr(), float(eps), flags,
                              wptr, wlen, stream_handle(ipos.device)), "calc_acc")


def accelerations(ipos: torch.Tensor, eps: float, jpos: torch.Tensor | None = None, *, potential: bool = False,
                  exact: bool = False) -> torch.Tensor:
    """Convenience: returns a new ``[Ni, 4]`` acceleration tensor."""
    jpos = ipos if jpos is None else jpos
    iacc = torch.empty_like(ipos)
    calc_acc(ipos.shape[0], ipos, iacc, jpos.shape[0], jpos, eps, potential=potential, exact=exact)
    return iacc


def kdk_update(pos: torch.Tensor | None, vel: torch.Tensor | None, acc: torch.Tensor, partials: torch.Tensor | None,
               nchunks: int, h_end: float, h_begin: float, dt: float, phases: int) -> None:
    """Fused K2 update (b2_kdk_update): reduce j-chunk partials, closing kick, opening kick + drift."""
    n = acc.shape[0]
    ptr = lambda t: t.data_ptr() if t is not None else None  # noqa: E731
    with on_device(acc.device):
        check(load().b2_kdk_update(n, ptr(pos), ptr(vel), acc.data_ptr(), ptr(partials), nchunks, float(h_end),
                                   float(h_begin), float(dt), phases, stream_handle(acc.device)), "kdk_update")


@dataclass
class Leapfrog:
    """Kick-drift-kick leapfrog of a self-gravitating system on one GPU.

    One step: ``v += a h; x += v dt; a = calc_acc(x); v += a h`` with
    ``h = dt/2``. Steady state is two launches per step (force, fused update).
    Up to 64 x SMs particles (9472 on a B200) the whole run is one persistent launch; between that and
    ``GRAPH_MAX_N`` particles the per-step launches are the overhead, so ``step(k)``
    (k >= 2) is captured once per k into a CUDA graph and replayed (``graphs=False``
    turns that off; the same kernels run either way, so the results are identical).
    """

    GRAPH_MIN_N = 9473
    GRAPH_MAX_N = 1 << 15

    pos: torch.Tensor
    vel: torch.Tensor
    eps: float
    dt: float
    potential: bool = False
    exact: bool = False
    graphs: bool = True

    def __post_init__(self) -> None:
        n = self.pos.shape[0]
        _particles(self.pos, n, "pos")
        _particles(self.vel, n, "vel")
        self.acc = torch.empty_like(self.pos)
        self._flags = _flags(self.potential, self.exact)
        self._ws = torch.empty(max(int(load().b2_leapfrog_workspace_bytes(n, self._flags)), 16),
                               dtype=torch.uint8, device=self.pos.device)
        self.steps = 0
        self._graphs: dict[int, torch.cuda.CUDAGraph] = {}
        self._run(0, init=True)

    def _run(self, nsteps: int, init: bool = False) -> None:
        n = self.pos.shape[0]
        flags = self._flags | (_lib.B2_INIT_ACC if init else 0)
        with on_device(self.pos.device):
            check(load().b2_leapfrog(n, self.pos.data_ptr(), self.vel.data_ptr(), self.acc.data_ptr(),
                                     float(self.eps), float(self.dt), int(nsteps), flags, self._ws.data_ptr(),
                                     self._ws.numel(), stream_handle(self.pos.device)), "leapfrog")

    def step(self, nsteps: int = 1) -> None:
        g = self._graph_for(nsteps)
        if g is not None:
            g.replay()
        else:
            self._run(nsteps)
        self.steps += nsteps

    def _graph_for(self, nsteps: int):
        """The captured ``b2_leapfrog(nsteps)`` for launch-bound sizes, else None."""
        n = self.pos.shape[0]
        if (not self.graphs or nsteps < 2 or not (self.GRAPH_MIN_N <= n <= self.GRAPH_MAX_N)
                or torch.cuda.is_current_stream_capturing()):
            return None
        g = self._graphs.get(nsteps)
        if g is None:
            try:
                g = torch.cuda.CUDAGraph()
                side = torch.cuda.Stream(self.pos.device)
                side.wait_stream(torch.cuda.current_stream(self.pos.device))
                with torch.cuda.graph(g, stream=side):
                    self._run(nsteps)  # recorded, not executed
                torch.cuda.current_stream(self.pos.device).wait_stream(side)
            except RuntimeError:  # capture refused: stay on direct launches
                self.graphs = False
                return None
            self._graphs[nsteps] = g
        return g

    def kernel_launches_per_step(self) -> int:
        return 2

    def synchronize(self) -> None:
        """Wait for the queued steps; raises SolomonError if a device-side wait gave up
        (the persistent small-N path exchanges positions between CTAs in the GPU)."""
        _lib.check_fault(self.pos.device, "Leapfrog.step")

    # ---- checkpoint / resume -----------------------------------
    def state_dict(self) -> dict:
        """Positions, velocities (synchronised: every step closes with its half-kick),
        accelerations a(pos) and the step count -- everything a resumed run needs."""
        return {"kind": "Leapfrog", "pos": self.pos.clone(), "vel": self.vel.clone(), "acc": self.acc.clone(),
                "eps": self.eps, "dt": self.dt, "potential": self.potential, "exact": self.exact,
                "steps": self.steps}

    def load_state_dict(self, sd: dict) -> None:
        if sd.get("kind") != "Leapfrog":
            raise ValueError(f"not a Leapfrog checkpoint: {sd.get('kind')!r}")
        if tuple(sd["pos"].shape) != tuple(self.pos.shape):
            raise ValueError(f"checkpoint holds {tuple(sd['pos'].shape)} particles, this run {tuple(self.pos.shape)}")
        if (sd["eps"], sd["dt"], sd["potential"], sd["exact"]) != (self.eps, self.dt, self.potential, self.exact):
            raise ValueError("checkpoint eps/dt/potential/exact differ from this run's")
        self.pos.copy_(sd["pos"])
        self.vel.copy_(sd["vel"])
        self.acc.copy_(sd["acc"])
        self.steps = int(sd["steps"])

    @classmethod
    def from_state_dict(cls, sd: dict, device: torch.device | str = "cuda") -> "Leapfrog":
        lf = cls(sd["pos"].to(device), sd["vel"].to(device), sd["eps"], sd["dt"], sd["potential"], sd["exact"])
        lf.load_state_dict(sd)
        return lf


def leapfrog_kdk(pos: torch.Tensor, vel: torch.Tensor, eps: float, dt: float, nsteps: int, *,
                 potential: bool = False, exact: bool = False):
    """Functional form: integrate copies of (pos, vel); returns (pos, vel, acc)."""
    lf = Leapfrog(pos.clone(), vel.clone(), eps, dt, potential, exact)
    lf.step(nsteps)
    return lf.pos, lf.vel, lf.acc


# ---------------------------------------------------------------------------
# Initial conditions (no reference counterpart). Generated on
# the host in FP64 with a fixed seed and cast to FP32 once, so the GPU run
# and the CPU oracle see identical inputs.

def plummer_numpy(n: int, seed: int = 42) -> tuple[np.ndarray, np.ndarray]:
    """Plummer sphere (Aarseth, Henon & Wielen 1974) in standard units (G = M = 1, E = -1/4).

    Returns float32 ``pos[n,4] = {x,y,z,m=1/n}`` and ``vel[n,4] = {vx,vy,vz,0}``,
    centre-of-mass frame. Radii from the inverted cumulative mass with
    X1 < 0.999 (truncation); speeds by von Neumann rejection on
    g(q) = q^2 (1 - q^2)^{7/2}; lengths scaled by 3*pi/16, velocities by
    sqrt(16 / (3*pi)).
    """
    rng = np.random.default_rng(seed)
    x1 = rng.uniform(0.0, 0.999, n)
    x1 = np.maximum(x1, 1e-10)
    r = 1.0 / np.sqrt(x1 ** (-2.0 / 3.0) - 1.0)

    def iso(mag: np.ndarray) -> np.ndarray:
        u = rng.uniform(-1.0, 1.0, mag.shape[0])
        phi = rng.uniform(0.0, 2.0 * np.pi, mag.shape[0])
        s = np.sqrt(1.0 - u * u)
        return mag[:, None] * np.stack([s * np.cos(phi), s * np.sin(phi), u], axis=1)

    xyz = iso(r)
    q = np.empty(n)
    todo = np.arange(n)
    while todo.size:
        qq = rng.uniform(0.0, 1.0, todo.size)
        gg = rng.uniform(0.0, 0.1, todo.size)
        ok = gg < qq * qq * (1.0 - qq * qq) ** 3.5
        q[todo[ok]] = qq[ok]
        todo = todo[~ok]
    ve = np.sqrt(2.0) * (1.0 + r * r) ** -0.25
    v = iso(q * ve)
    a = 3.0 * np.pi / 16.0
    xyz *= a
    v /= math.sqrt(a)
    xyz -= xyz.mean(axis=0)
    v -= v.mean(axis=0)
    pos = np.empty((n, 4), np.float32)
    vel = np.zeros((n, 4), np.float32)
    pos[:, :3] = xyz
    pos[:, 3] = 1.0 / n
    vel[:, :3] = v
    return pos, vel


def uniform_numpy(n: int, seed: int = 42, half_width: float = 1.0) -> tuple[np.ndarray, np.ndarray]:
    """Uniform cube [-w, w]^3, masses 1/n, at rest."""
    rng = np.random.default_rng(seed)
    pos = np.empty((n, 4), np.float32)
    pos[:, :3] = rng.uniform(-half_width, half_width, (n, 3))
    pos[:, 3] = 1.0 / n
    return pos, np.zeros((n, 4), np.float32)


def plummer(n: int, seed: int = 42, device: torch.device | str = "cuda") -> tuple[torch.Tensor, torch.Tensor]:
    p, v = plummer_numpy(n, seed)
    return torch.from_numpy(p).to(device), torch.from_numpy(v).to(device)


def uniform(n: int, seed: int = 42, device: torch.device | str = "cuda") -> tuple[torch.Tensor, torch.Tensor]:
    p, v = uniform_numpy(n, seed)
    return torch.from_numpy(p).to(device), torch.from_numpy(v).to(device)


def energy(pos: torch.Tensor, vel: torch.Tensor, acc_pot: torch.Tensor, eps: float) -> tuple[float, float]:
    """(kinetic, potential) energy; ``acc_pot`` from calc_acc(..., potential=True).

    The reference's potential sum includes the self term m_i/eps (j = i is
    not skipped, listing_nbody.c:8); it is removed here. Diagnostic only.
    """
    m = pos[:, 3].double()
    ke = 0.5 * (m * (vel[:, :3].double() ** 2).sum(dim=1)).sum()
    pot = acc_pot[:, 3].double() - m / float(eps)
    pe = -0.5 * (m * pot).sum()
    return float(ke), float(pe)
