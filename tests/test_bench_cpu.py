"""CPU: bench.py's reference arm (no GPU needed) prints one well-formed JSON line."""
from __future__ import annotations

import json
import pathlib
import subprocess
import sys

import pytest

ROOT = pathlib.Path(__file__).resolve().parents[1]


def test_reference_arm_json_line(tmp_path):
    import oracle

    if not oracle.Reference.available("fast"):
        pytest.skip("oracle/_ref not built")
    results = tmp_path / "results.jsonl"
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1", "--warmup", "0",
                          "--cpu-seconds", "0.3", "--n", "16384", "--grid", "64", "--results", str(results)],
                         cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1  # stdout is the JSON line and nothing else
    assert results.read_text().splitlines() == lines  # --results appends the same line
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["unit"] == "Ginteractions/s" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert d["secondary"]["diffusion"]["value"] > 0


def test_clock_sampler_parses_nvidia_smi_csv(tmp_path):
    sys.path.insert(0, str(ROOT))
    import bench

    s = bench.ClockSampler(0)
    s.file = open(tmp_path / "c.csv", "w+")
    s.file.write("0, 1965, 1965, 700.1, 0x0, Not Active, Not Active, Not Active, Not Active\n"
                 "0, 1800, 1965, 990.0, 0x4, Not Active, Not Active, Not Active, Active\n"
                 "0, 1965, 1965, 800.0, 0x0, Not Active, Not Active, Not Active, Not Active\n")
    s.file.flush()

    class _P:
        def terminate(self):
            pass

        def wait(self, timeout=None):
            return 0

    s.proc = _P()
    rec = s.stop()
    assert rec == {"sm_mhz": 1965.0, "sm_max_mhz": 1965.0, "reasons": ["sw_power_cap"], "samples": 3}


def test_parity_checkers_accept_the_reference_and_reject_perturbations():
    """bench.py's full-size parity helpers (run as checkers outside the timed regions): the
    reference's own output passes, a perturbed one fails."""
    import numpy as np

    import oracle

    if not oracle.Reference.available("ieee"):
        pytest.skip("oracle/_ref not built")
    sys.path.insert(0, str(ROOT))
    import bench
    from paper_2411_18889_b200.nbody import plummer_numpy

    pos, _ = plummer_numpy(2048, 3)
    acc = oracle.Reference("ieee").calc_acc(pos, pos, bench.EPS)
    ok = bench.nbody_sample_parity(pos, acc, n_sample=128)
    assert ok["ok"] and ok["relL2_acc"] == 0.0
    bad = acc.copy()
    bad[:, :3] *= 1.001
    assert not bench.nbody_sample_parity(pos, bad, n_sample=128)["ok"]

    args = (0.03, 0.02, 0.025, 2e-5, 1.0)
    f0 = np.random.default_rng(1).random((6, 7, 8), dtype=np.float32)
    want = oracle.Reference("ieee").diffusion_run(f0, 3, *args)
    assert bench.diffusion_parity(f0, want, 3, args)["bit_identical"]
    off = want.copy()
    off[2, 3, 4] = np.nextafter(off[2, 3, 4], np.float32(2))
    r = bench.diffusion_parity(f0, off, 3, args)
    assert not r["bit_identical"] and r["relL2"] > 0


def test_compact_line_keeps_the_contract_keys():
    """The driver keeps only the tail of stdout: compact() of a real full record (the committed
    round-2 detail file) carries every contract key in a short line."""
    sys.path.insert(0, str(ROOT))
    import bench

    full = json.loads((ROOT / "profiles" / "r02" / "bench_detail_r02k.json").read_text())
    line = json.dumps(bench.compact(full))
    assert len(line) < 4096
    d = json.loads(line)
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "gpu_launches", "clocks", "roofline", "cpu_baseline", "e2e"):
        assert k in d, k
    assert {"bound", "achieved", "peak", "unit", "frac", "traffic"} <= set(d["roofline"])
    assert {"value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"} <= set(d["e2e"])
    assert {"value", "unit", "cores", "kind", "sample"} <= set(d["cpu_baseline"])
    sec = d["secondary"]
    assert sec["diffusion"]["roofline"]["bound"] == "hbm" and sec["diffusion"]["bit_identical"] is True
    assert sec["diffusion_run"]["bit_identical"] is True and sec["nbody_uniform"]["ok"] is True
    assert "config0" in sec and "config1" in sec
