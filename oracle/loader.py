"""ctypes loaders for the oracle libraries -- TEST INFRASTRUCTURE ONLY."""
from __future__ import annotations

import ctypes
import os
import pathlib

import numpy as np

HERE = pathlib.Path(__file__).resolve().parent
_f32p = ctypes.POINTER(ctypes.c_float)


def cpu_isa() -> str:
    """'native' when the host has the AVX-512 the native build assumes, else 'v3'."""
    try:
        flags = pathlib.Path("/proc/cpuinfo").read_text()
    except OSError:
        return "v3"
    return "native" if ("avx512f" in flags and "avx512vl" in flags) else "v3"


def _ptr(a: np.ndarray):
    assert a.dtype == np.float32 and a.flags.c_contiguous
    return a.ctypes.data_as(_f32p)


def _load(path: pathlib.Path) -> ctypes.CDLL:
    if not path.exists():
        raise FileNotFoundError(f"{path} missing: run `make -C oracle` (or __graft_entry__.build())")
    return ctypes.CDLL(str(path))


def diffusion_coeffs(dx, dy, dz, dt, kappa):
    """(cc, ce, cn, ct) exactly as listing_diffusion.c:6-9 computes them in FP32."""
    f = np.float32
    kd = f(kappa) * f(dt)
    ce = kd / (f(dx) * f(dx))
    cn = kd / (f(dy) * f(dy))
    ct = kd / (f(dz) * f(dz))
    cc = f(1.0) - (((((ce + ce) + cn) + cn) + ct) + ct)
    return f(cc), f(ce), f(cn), f(ct)


class _Base:
    threads: int = os.cpu_count() or 1

    def calc_acc(self, ipos: np.ndarray, jpos: np.ndarray, eps: float, potential: bool = False) -> np.ndarray:
        ipos = np.ascontiguousarray(ipos, dtype=np.float32)
        jpos = np.ascontiguousarray(jpos, dtype=np.float32)
        out = np.zeros_like(ipos)
        self._calc_acc(ipos.shape[0], _ptr(ipos), _ptr(out), jpos.shape[0], _ptr(jpos),
                       ctypes.c_float(eps), int(potential))
        return out

    def diffusion3d(self, f: np.ndarray, dx, dy, dz, dt, kappa) -> np.ndarray:
        f = np.ascontiguousarray(f, dtype=np.float32)
        nx, ny, nz = f.shape
        fn = np.empty_like(f)
        self._diffusion3d(nx, ny, nz, ctypes.c_float(dx), ctypes.c_float(dy), ctypes.c_float(dz),
                          ctypes.c_float(dt), ctypes.c_float(kappa), _ptr(f), _ptr(fn))
        return fn

    def diffusion_run(self, f: np.ndarray, steps: int, dx, dy, dz, dt, kappa) -> np.ndarray:
        a = np.ascontiguousarray(f, dtype=np.float32).copy()
        for _ in range(steps):
            a = self.diffusion3d(a, dx, dy, dz, dt, kappa)
        return a


class Restatement(_Base):
    """Our C restatement (solomon_oracle.c)."""

    def __init__(self, isa: str | None = None):
        self.lib = _load(HERE / f"liboracle_{isa or cpu_isa()}.so")
        L = self.lib
        L.oracle_calc_acc.argtypes = [ctypes.c_int, _f32p, _f32p, ctypes.c_int, _f32p, ctypes.c_float, ctypes.c_int]
        L.oracle_diffusion3d.argtypes = [ctypes.c_int] * 3 + [ctypes.c_float] * 5 + [_f32p, _f32p]
        L.oracle_leapfrog.argtypes = [ctypes.c_int, _f32p, _f32p, _f32p, ctypes.c_float, ctypes.c_float,
                                      ctypes.c_int, ctypes.c_int]
        L.oracle_calc_acc_partials.argtypes = [ctypes.c_int, _f32p, ctypes.c_int, _f32p, ctypes.c_float,
                                               ctypes.c_int, ctypes.c_int, _f32p]
        L.oracle_kdk_update.argtypes = [ctypes.c_int, _f32p, _f32p, _f32p, _f32p, ctypes.c_int, ctypes.c_float,
                                        ctypes.c_float, ctypes.c_float, ctypes.c_int]
        L.oracle_calc_acc_f64.argtypes = [ctypes.c_int, _f32p, ctypes.POINTER(ctypes.c_double), ctypes.c_int, _f32p,
                                          ctypes.c_float]
        self._calc_acc = L.oracle_calc_acc
        self._diffusion3d = L.oracle_diffusion3d

    def calc_acc_f64(self, ipos, jpos, eps) -> np.ndarray:
        """FP64 yardstick (exact 1/sqrt, double sums): float64[Ni, 4], .w = the potential sum."""
        ipos = np.ascontiguousarray(ipos, dtype=np.float32)
        jpos = np.ascontiguousarray(jpos, dtype=np.float32)
        out = np.zeros((ipos.shape[0], 4), np.float64)
        self.lib.oracle_calc_acc_f64(ipos.shape[0], _ptr(ipos), out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                     jpos.shape[0], _ptr(jpos), ctypes.c_float(eps))
        return out

    def calc_acc_partials(self, ipos, jpos, eps, chunk, potential=False, out=None):
        ipos = np.ascontiguousarray(ipos, dtype=np.float32)
        jpos = np.ascontiguousarray(jpos, dtype=np.float32)
        nch = (jpos.shape[0] + chunk - 1) // chunk
        if out is None:
            out = np.empty((nch * ipos.shape[0], 4), np.float32)
        self.lib.oracle_calc_acc_partials(ipos.shape[0], _ptr(ipos), jpos.shape[0], _ptr(jpos), ctypes.c_float(eps),
                                          int(potential), int(chunk), _ptr(out))
        return out

    def kdk_update(self, pos, vel, acc, partials, nchunks, h_end, h_begin, dt, phases):
        """In place on float32 C-contiguous arrays (None allowed where the phase does not use it)."""
        p = lambda a: _ptr(a) if a is not None else None  # noqa: E731
        self.lib.oracle_kdk_update(acc.shape[0], p(pos), p(vel), _ptr(acc), p(partials), int(nchunks),
                                   ctypes.c_float(h_end), ctypes.c_float(h_begin), ctypes.c_float(dt), int(phases))

    def leapfrog(self, pos, vel, eps, dt, nsteps, potential=False):
        """Returns (pos, vel, acc) after ``nsteps`` KDK steps (spec: solomon_oracle.c)."""
        pos = np.ascontiguousarray(pos, dtype=np.float32).copy()
        vel = np.ascontiguousarray(vel, dtype=np.float32).copy()
        acc = self.calc_acc(pos, pos, eps, potential)
        self.lib.oracle_leapfrog(pos.shape[0], _ptr(pos), _ptr(vel), _ptr(acc), ctypes.c_float(eps),
                                 ctypes.c_float(dt), int(nsteps), int(potential))
        return pos, vel, acc


class Reference(_Base):
    """The reference's own listings, fallback-lowered and g++-compiled (oracle/_ref)."""

    def __init__(self, variant: str = "ieee", isa: str | None = None):
        self.variant = variant
        self.lib = _load(HERE / "_ref" / f"libref_{variant}_{isa or cpu_isa()}.so")
        L = self.lib
        L.ref_calc_acc.argtypes = [ctypes.c_int, _f32p, _f32p, ctypes.c_int, _f32p, ctypes.c_float, ctypes.c_int]
        L.ref_diffusion3d.argtypes = [ctypes.c_int] * 3 + [ctypes.c_float] * 5 + [_f32p, _f32p]
        self._calc_acc = L.ref_calc_acc
        self._diffusion3d = L.ref_diffusion3d

    @staticmethod
    def available(variant: str = "ieee") -> bool:
        return (HERE / "_ref" / f"libref_{variant}_{cpu_isa()}.so").exists()
