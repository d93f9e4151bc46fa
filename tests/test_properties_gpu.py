"""Property-based parity on the GPU (the reference's property-test pattern,
pkg/tests/test_properties.py:56-146: seeded hypothesis cases with a fixed
max_examples, checked against an independent oracle).

Random shapes and step counts drive every dispatch path of the diffusion time
loop (shared-memory-resident bricks, cooperative multi-step, two steps per HBM
pass, single-step march / direct / generic kernels) and of the n-body force
(exact, fast large-tile, medium and small variants, ragged chunks, Ni != Nj);
each case is compared with the oracle restatement: bit for bit for diffusion
and exact n-body, within the stated tolerance for fast n-body.
"""
from __future__ import annotations

import numpy as np
import pytest

from conftest import bits_equal, rel_l2

torch = pytest.importorskip("torch")
hyp = pytest.importorskip("hypothesis")
from hypothesis import HealthCheck, given, settings  # noqa: E402
from hypothesis import strategies as st  # noqa: E402

pytestmark = pytest.mark.gpu

SETTINGS = settings(max_examples=100, deadline=None, derandomize=True,
                    suppress_health_check=[HealthCheck.function_scoped_fixture, HealthCheck.too_slow])


@pytest.fixture(scope="module")
def b2():
    import paper_2411_18889_b200 as b2

    b2.load()
    return b2


@SETTINGS
@given(nx=st.integers(1, 70), ny=st.integers(1, 70), nz4=st.integers(1, 48), nz_off=st.sampled_from([0, 0, 0, 1, 3]),
       steps=st.integers(0, 7), seed=st.integers(0, 2 ** 16))
def test_diffusion_run_any_shape_bit_identical(b2, restatement, nx, ny, nz4, nz_off, steps, seed):
    nz = 4 * nz4 + nz_off  # nz % 4 != 0 exercises the generic kernel
    args = (0.031, 0.027, 0.022, 2e-5, 1.0)
    f0 = np.random.default_rng(seed).random((nx, ny, nz), dtype=np.float32)
    want = restatement.diffusion_run(f0, steps, *args)
    got = b2.Diffusion3D(torch.from_numpy(f0).cuda(), *args).run(steps).cpu().numpy()
    assert bits_equal(got, want)


@settings(max_examples=40, deadline=None, derandomize=True,
          suppress_health_check=[HealthCheck.function_scoped_fixture, HealthCheck.too_slow])
@given(g=st.sampled_from([128, 256, 512]), ny=st.integers(9, 300), nx=st.integers(2, 40), steps=st.integers(1, 5),
       seed=st.integers(0, 2 ** 16))
def test_diffusion_run_two_steps_per_pass_shapes(b2, restatement, g, ny, nx, steps, seed):
    """Row pitches the two-steps-per-pass kernel takes, ragged tiles in j, short i ranges."""
    args = (0.031, 0.027, 0.022, 2e-5, 1.0)
    f0 = np.random.default_rng(seed).random((nx, ny, g), dtype=np.float32)
    want = restatement.diffusion_run(f0, steps, *args)
    got = b2.Diffusion3D(torch.from_numpy(f0).cuda(), *args).run(steps).cpu().numpy()
    assert bits_equal(got, want)


@SETTINGS
@given(ni=st.integers(1, 3000), nj=st.integers(1, 9000), potential=st.booleans(), seed=st.integers(0, 2 ** 16))
def test_calc_acc_any_sizes(b2, restatement, ni, nj, potential, seed):
    rng = np.random.default_rng(seed)
    jpos = np.empty((nj, 4), np.float32)
    jpos[:, :3] = rng.uniform(-1, 1, (nj, 3))
    jpos[:, 3] = rng.uniform(0.5, 1.5, nj) / nj
    ipos = jpos[rng.integers(0, nj, ni)].copy()
    eps = 2.0 ** -6
    want = restatement.calc_acc(ipos, jpos, eps, potential=potential)
    ip, jp = torch.from_numpy(ipos).cuda(), torch.from_numpy(jpos).cuda()
    out = torch.empty_like(ip)
    b2.calc_acc(ni, ip, out, nj, jp, eps, potential=potential, exact=True)
    assert bits_equal(out.cpu().numpy(), want)
    b2.calc_acc(ni, ip, out, nj, jp, eps, potential=potential)
    got = out.cpu().numpy()
    assert rel_l2(got[:, :3], want[:, :3]) < 1e-5
    if potential:
        assert rel_l2(got[:, 3], want[:, 3]) < 1e-5


@settings(max_examples=30, deadline=None, derandomize=True,
          suppress_health_check=[HealthCheck.function_scoped_fixture, HealthCheck.too_slow])
@given(n=st.integers(2, 9472), steps=st.integers(0, 4), potential=st.booleans(), seed=st.integers(0, 2 ** 16))
def test_leapfrog_small_n_tracks_oracle(b2, restatement, n, steps, potential, seed):
    """The persistent small-N leapfrog (and the two-kernel path it must equal) against the oracle KDK."""
    pos, vel = b2.plummer_numpy(n, seed)
    wp, wv, _ = restatement.leapfrog(pos, vel, 2.0 ** -6, 2.0 ** -7, steps, potential=potential)
    p, v, _ = b2.leapfrog_kdk(torch.from_numpy(pos).cuda(), torch.from_numpy(vel).cuda(), 2.0 ** -6, 2.0 ** -7,
                              steps, potential=potential)
    assert rel_l2(p.cpu().numpy()[:, :3], wp[:, :3]) < 1e-5
    assert rel_l2(v.cpu().numpy()[:, :3], wv[:, :3]) < 1e-4 + 1e-4 * (np.linalg.norm(wv[:, :3]) == 0)
