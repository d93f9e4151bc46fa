"""Compiled callers of the drop-in: a C++ driver with its OWN ``struct float4`` and a C99 driver
with its own ``float4`` typedef, both calling the reference signatures unchanged
(``listing_nbody.c:1``, ``listing_diffusion.c:5``) and linked against ``-lsolomon_b200``.

CPU: both compile and link warning-free (-Werror) against include/solomon_b200.h, and on a
GPU-less box the drop-in reports the CUDA error through b2_last_error instead of crashing.
GPU: their outputs match the oracle (calc_acc_exact and diffusion3d bit for bit, calc_acc
within the fast path's tolerance).
"""
from __future__ import annotations

import pathlib
import shutil
import subprocess

import numpy as np
import pytest

from conftest import bits_equal, rel_l2

ROOT = pathlib.Path(__file__).resolve().parents[1]
LIBDIR = ROOT / "paper_2411_18889_b200" / "lib"
DRIVERS = ROOT / "tests" / "drivers"


def _build(tmp_path, which: str) -> pathlib.Path:
    if not (LIBDIR / "libsolomon_b200.so").exists():
        pytest.skip("library not built")
    exe = tmp_path / f"driver_{which}"
    if which == "cpp":
        cmd = [shutil.which("g++") or "g++", "-std=c++17", "-O2", "-Wall", "-Wextra", "-Werror",
               str(DRIVERS / "driver_cpp.cpp")]
    else:
        cmd = [shutil.which("gcc") or "gcc", "-std=c99", "-O2", "-Wall", "-Wextra", "-Werror", "-pedantic",
               str(DRIVERS / "driver_c.c")]
    cmd += [f"-I{ROOT / 'include'}", f"-L{LIBDIR}", "-lsolomon_b200", f"-Wl,-rpath,{LIBDIR}", "-o", str(exe)]
    out = subprocess.run(cmd, capture_output=True, text=True)
    assert out.returncode == 0, out.stderr
    return exe


def _inputs(tmp_path, n=700, shape=(12, 10, 20)):
    from paper_2411_18889_b200.nbody import plummer_numpy

    pos, _ = plummer_numpy(n, 11)
    f = np.random.default_rng(5).random(shape, dtype=np.float32)
    par = np.array([2.0 ** -6, 0.1, 0.11, 0.09, 1e-3, 1.0], np.float32)
    path = tmp_path / "in.bin"
    with open(path, "wb") as fh:
        fh.write(np.array([n, *shape], np.int32).tobytes())
        fh.write(par.tobytes())
        fh.write(pos.tobytes())
        fh.write(f.tobytes())
    return path, pos, f, par


@pytest.mark.parametrize("which", ["cpp", "c"])
def test_driver_compiles_links_and_reports_errors_without_gpu(tmp_path, which):
    import torch

    exe = _build(tmp_path, which)
    if torch.cuda.is_available():
        pytest.skip("GPU present: see test_driver_results_match_oracle")
    path, *_ = _inputs(tmp_path, n=64, shape=(4, 4, 8))
    out = subprocess.run([str(exe), str(path), str(tmp_path / "out.bin")], capture_output=True, text=True, timeout=120)
    assert out.returncode == 3, (out.returncode, out.stderr)  # the error reached the caller (b2_last_error)
    assert "solomon_b200: calc_acc failed" in out.stderr  # ... and stderr, like report() promises
    assert "out of device memory" not in out.stderr  # the real CUDA error, not a generic ENOMEM


@pytest.mark.gpu
@pytest.mark.parametrize("which", ["cpp", "c"])
def test_driver_results_match_oracle(tmp_path, which, restatement):
    exe = _build(tmp_path, which)
    n, shape = 700, (12, 10, 20)
    path, pos, f, par = _inputs(tmp_path, n, shape)
    out = subprocess.run([str(exe), str(path), str(tmp_path / "out.bin")], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    raw = np.fromfile(tmp_path / "out.bin", dtype=np.float32)
    acc, exact, pot = (raw[k * 4 * n:(k + 1) * 4 * n].reshape(n, 4) for k in range(3))
    fn = raw[12 * n:].reshape(shape)
    eps = float(par[0])
    want = restatement.calc_acc(pos, pos, eps)
    want_pot = restatement.calc_acc(pos, pos, eps, potential=True)
    assert bits_equal(exact, want)                      # calc_acc_exact: the reference's bits
    assert rel_l2(acc[:, :3], want[:, :3]) < 1e-5       # fast path tolerance
    assert rel_l2(pot[:, 3], want_pot[:, 3]) < 1e-5
    assert bits_equal(fn, restatement.diffusion3d(f, *(float(x) for x in par[1:])))
