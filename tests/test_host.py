"""CPU: host-side logic -- initial conditions, coefficients, bindings, no-fallback behaviour."""
from __future__ import annotations

import numpy as np
import pytest
import torch

import paper_2411_18889_b200 as b2


def test_plummer_standard_units():
    """Henon units: virial ratio ~1/2, total energy ~ -1/4, centre-of-mass frame, masses 1/N."""
    import oracle

    n = 8192
    pos, vel = b2.plummer_numpy(n, 42)
    assert pos.dtype == np.float32 and pos.shape == (n, 4) and vel.shape == (n, 4)
    assert np.allclose(pos[:, 3], 1.0 / n)
    assert np.all(vel[:, 3] == 0)
    m = pos[:, 3].astype(np.float64)
    assert np.abs((m[:, None] * pos[:, :3]).sum(0)).max() < 1e-6
    assert np.abs((m[:, None] * vel[:, :3]).sum(0)).max() < 1e-6
    eps = 1e-4
    acc = oracle.Restatement().calc_acc(pos, pos, eps, potential=True).astype(np.float64)
    ke = 0.5 * (m * (vel[:, :3].astype(np.float64) ** 2).sum(1)).sum()
    pe = -0.5 * (m * (acc[:, 3] - m / eps)).sum()
    assert ke + pe == pytest.approx(-0.25, abs=0.02)
    assert 2 * ke / -pe == pytest.approx(1.0, abs=0.06)


def test_plummer_deterministic_and_truncated():
    a, _ = b2.plummer_numpy(1000, 7)
    b, _ = b2.plummer_numpy(1000, 7)
    c, _ = b2.plummer_numpy(1000, 8)
    assert np.array_equal(a, b) and not np.array_equal(a, c)
    r = np.linalg.norm(a[:, :3], axis=1)
    assert r.max() < 3 * np.pi / 16 / np.sqrt(0.999 ** (-2 / 3) - 1) + 0.5  # X1 < 0.999 truncation


def test_uniform_cube():
    p, v = b2.uniform_numpy(1000, 3, half_width=2.0)
    assert np.abs(p[:, :3]).max() <= 2.0 and np.all(v == 0) and np.allclose(p[:, 3], 1e-3)


def test_coefficients_follow_listing():
    c = b2.coefficients(0.1, 0.2, 0.4, 1e-3, 2.0)
    kd = np.float32(2.0) * np.float32(1e-3)
    assert c["ce"] == np.float32(kd / np.float32(np.float32(0.1) * np.float32(0.1)))
    assert c["cw"] == c["ce"] and c["cs"] == c["cn"] and c["cb"] == c["ct"]
    s = np.float32(0)
    for k in ("ce", "cw", "cn", "cs", "ct", "cb"):
        s = np.float32(s + np.float32(c[k]))
    assert c["cc"] == np.float32(1) - s


def test_no_cpu_fallback():
    """Compute calls on CPU tensors raise instead of silently running elsewhere."""
    with pytest.raises(b2.SolomonError):
        b2.accelerations(torch.zeros(8, 4), 0.1)
    f = torch.zeros(4, 4, 4)
    with pytest.raises(b2.SolomonError):
        b2.diffusion3d(4, 4, 4, 1.0, 1.0, 1.0, 0.1, 1.0, f, torch.zeros_like(f))


def test_missing_library_fails_loudly(tmp_path):
    from paper_2411_18889_b200 import _lib

    with pytest.raises(_lib.SolomonError):
        _lib.load(tmp_path / "nope.so")


def test_package_does_not_import_oracle():
    """The product path never routes through the checker."""
    import pathlib
    import re

    pkg = pathlib.Path(b2.__file__).parent
    for py in pkg.rglob("*.py"):
        assert not re.search(r"^\s*(import|from)\s+oracle", py.read_text(), flags=re.M), py
    for cu in (pkg / "csrc").glob("*.c*"):
        assert "oracle" not in cu.read_text().lower() or cu.name == "probe.cu", cu


def test_residency_requires_mapping():
    from paper_2411_18889_b200 import residency as R

    a = np.zeros(8, np.float32)
    assert not R.is_present(a)
    with pytest.raises(b2.SolomonError):
        R.present(a)
    with pytest.raises(b2.SolomonError):
        R.free_from_device(a)
    with pytest.raises(b2.SolomonError):  # DATA_ACCESS_BY_HOST (use_device) needs a present array
        with R.data_access_by_host(a):
            pass
    if not torch.cuda.is_available():
        with pytest.raises(b2.SolomonError):
            R.malloc_on_device(a)


def test_sharded_checkpoint_path_needs_rank_placeholder(tmp_path):
    """at world size > 1 every rank writing one path would lose shards silently."""
    import types

    from paper_2411_18889_b200 import checkpoint

    slab = types.SimpleNamespace(rank=1, world=2)
    with pytest.raises(ValueError, match="rank"):
        checkpoint._rank_path(tmp_path / "ck.pt", slab)
    assert checkpoint._rank_path(str(tmp_path / "ck.{rank}.pt"), slab).name == "ck.1.pt"
    shard = types.SimpleNamespace(plan=types.SimpleNamespace(rank=3, world=4))
    with pytest.raises(ValueError):
        checkpoint._rank_path(tmp_path / "ck.pt", shard)
    assert checkpoint._rank_path(str(tmp_path / "ck.{rank}.pt"), shard).name == "ck.3.pt"
    single = types.SimpleNamespace()
    assert checkpoint._rank_path(tmp_path / "ck.pt", single).name == "ck.pt"
