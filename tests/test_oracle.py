"""CPU: pin the oracle before trusting it (runs without a GPU).

* the C restatement (oracle/solomon_oracle.c) == the golden vectors, bit for bit;
* the reference's own build (oracle/_ref, when present) == the golden vectors;
* restatement == reference build on fresh seeded inputs (both ISAs);
* physics properties that need no oracle (SURVEY.md §4 carry-over).

Mirrors the reference's golden-row and parity tests (pkg/tests/test_conformance.py:17-22,
pkg/tests/test_scan_impls.py:43-55: 2000 random cases, seed 1337).
"""
from __future__ import annotations

import numpy as np
import pytest

from conftest import bits_equal, rel_l2

NBODY = ["plummer256", "uniform300", "plummer1", "coincident5"]
DIFF = ["cube16", "aniso_12x20x24", "ragged_7x5x9", "thin_1x3x8", "line_2x1x40"]


@pytest.mark.parametrize("case", NBODY)
@pytest.mark.parametrize("potential", [False, True])
def test_restatement_matches_golden_nbody(restatement, golden, case, potential):
    pos = golden[f"nbody/{case}/pos"]
    eps = float(golden[f"nbody/{case}/eps"])
    want = golden[f"nbody/{case}/acc_pot" if potential else f"nbody/{case}/acc"]
    assert bits_equal(restatement.calc_acc(pos, pos, eps, potential), want)


def test_restatement_matches_golden_subset(restatement, golden):
    got = restatement.calc_acc(golden["nbody/subset/ipos"], golden["nbody/subset/jpos"],
                               float(golden["nbody/subset/eps"]))
    assert bits_equal(got, golden["nbody/subset/acc"])


@pytest.mark.parametrize("case", DIFF)
def test_restatement_matches_golden_diffusion(restatement, golden, case):
    params = [float(v) for v in golden[f"diff/{case}/params"]]
    got = restatement.diffusion_run(golden[f"diff/{case}/f0"], int(golden[f"diff/{case}/steps"]), *params)
    assert bits_equal(got, golden[f"diff/{case}/f"])


@pytest.mark.parametrize("case", NBODY)
def test_reference_build_reproduces_golden(reference, golden, case):
    pos = golden[f"nbody/{case}/pos"]
    eps = float(golden[f"nbody/{case}/eps"])
    assert bits_equal(reference.calc_acc(pos, pos, eps), golden[f"nbody/{case}/acc"])


@pytest.mark.parametrize("case", DIFF)
def test_reference_build_reproduces_golden_diffusion(reference, golden, case):
    params = [float(v) for v in golden[f"diff/{case}/params"]]
    got = reference.diffusion_run(golden[f"diff/{case}/f0"], int(golden[f"diff/{case}/steps"]), *params)
    assert bits_equal(got, golden[f"diff/{case}/f"])


@pytest.mark.parametrize("isa", ["native", "v3"])
def test_restatement_vs_reference_random(reference, isa):
    """Seeded random cases (the reference's parity-test style), both ISA builds."""
    import oracle

    if isa == "native" and oracle.cpu_isa() != "native":
        pytest.skip("host lacks AVX-512")
    rs = oracle.Restatement(isa)
    ref = oracle.Reference("ieee", isa)
    rng = np.random.default_rng(1337)
    for trial in range(20):
        n = int(rng.integers(1, 200))
        pos = rng.standard_normal((n, 4)).astype(np.float32)
        pos[:, 3] = rng.random(n).astype(np.float32)
        eps = float(rng.uniform(1e-3, 0.5))
        pot = bool(trial % 2)
        assert bits_equal(rs.calc_acc(pos, pos, eps, pot), ref.calc_acc(pos, pos, eps, pot))
        shape = tuple(int(v) for v in rng.integers(1, 14, 3))
        f = rng.random(shape, dtype=np.float32)
        params = tuple(float(v) for v in rng.uniform(0.05, 1.0, 3)) + (float(rng.uniform(1e-4, 1e-2)), 1.0)
        assert bits_equal(rs.diffusion3d(f, *params), ref.diffusion3d(f, *params))


def test_fast_reference_build_is_close(golden):
    """The -Ofast build (bench timing only) stays within FP32 tolerance of the IEEE build."""
    import oracle

    if not oracle.Reference.available("fast"):
        pytest.skip("oracle/_ref not built")
    fast = oracle.Reference("fast")
    pos = golden["nbody/plummer256/pos"]
    got = fast.calc_acc(pos, pos, float(golden["nbody/plummer256/eps"]))
    assert rel_l2(got, golden["nbody/plummer256/acc"]) < 1e-5


# ---- physics properties of the oracle itself ---------------------------------

def test_self_term_contributes_zero_acceleration(restatement):
    pos = np.array([[0.3, -0.2, 0.1, 2.0]], np.float32)
    acc = restatement.calc_acc(pos, pos, 0.1, potential=True)
    assert np.all(acc[0, :3] == 0)
    assert acc[0, 3] == pytest.approx(2.0 / 0.1, rel=1e-6)  # m / eps: the included j = i term


def test_pairwise_antisymmetry_and_momentum(restatement):
    from paper_2411_18889_b200.nbody import plummer_numpy

    pos, _ = plummer_numpy(512, 3)
    acc = restatement.calc_acc(pos, pos, 2.0 ** -6).astype(np.float64)
    m = pos[:, 3].astype(np.float64)
    net = (m[:, None] * acc[:, :3]).sum(0)
    assert np.all(np.abs(net) < 1e-5 * (m[:, None] * np.abs(acc[:, :3])).sum())


def test_two_body_analytic(restatement):
    eps = 0.05
    pos = np.array([[0, 0, 0, 1.0], [1.5, 0, 0, 2.0]], np.float32)
    acc = restatement.calc_acc(pos, pos, eps)
    expect = 2.0 * 1.5 / (1.5 ** 2 + eps ** 2) ** 1.5
    assert acc[0, 0] == pytest.approx(expect, rel=1e-6)
    assert acc[1, 0] == pytest.approx(-1.0 * 1.5 / (1.5 ** 2 + eps ** 2) ** 1.5, rel=1e-6)


def test_diffusion_conserves_mass_and_constant(restatement):
    rng = np.random.default_rng(2)
    f = rng.random((10, 11, 12), dtype=np.float32)
    args = (0.1, 0.1, 0.1, 1e-3, 1.0)
    out = restatement.diffusion_run(f, 20, *args)
    assert abs(out.sum(dtype=np.float64) - f.sum(dtype=np.float64)) / f.sum(dtype=np.float64) < 1e-5
    c = np.full((6, 7, 8), 0.25, np.float32)
    assert np.allclose(restatement.diffusion3d(c, *args), 0.25, rtol=0, atol=1e-7)


def test_leapfrog_restatement_time_reversible(restatement):
    from paper_2411_18889_b200.nbody import plummer_numpy

    pos, vel = plummer_numpy(256, 8)
    eps, dt = 2.0 ** -6, 2.0 ** -8
    p1, v1, _ = restatement.leapfrog(pos, vel, eps, dt, 8)
    p2, v2, _ = restatement.leapfrog(p1, -v1, eps, dt, 8)
    assert rel_l2(p2[:, :3], pos[:, :3]) < 1e-5
    assert rel_l2(-v2[:, :3], vel[:, :3]) < 1e-4


def test_f64_yardstick_and_reference_error_growth(restatement, reference):
    """The FP64 yardstick (calc_acc_f64) agrees with the reference's IEEE build to the latter's
    own FP32 error (~1e-6 at N=4096), and that error GROWS with N (sequential j-sum,
    listing_nbody.c:8-24) -- why large-N parity is judged against FP64."""
    from paper_2411_18889_b200.nbody import plummer_numpy

    errs = []
    for n in (4096, 65536):
        pos, _ = plummer_numpy(n, 42)
        sample = np.ascontiguousarray(pos[:: n // 64])
        exact = restatement.calc_acc_f64(sample, pos, 2.0 ** -6)[:, :3]
        ref = reference.calc_acc(sample, pos, 2.0 ** -6)[:, :3]
        errs.append(float(np.linalg.norm(ref - exact) / np.linalg.norm(exact)))
    assert errs[0] < 5e-6
    assert errs[1] > errs[0]
