"""Generate the golden vectors in tests/golden/ from the REFERENCE ITSELF.

The reference has no numeric golden vectors for its two kernels (its tests
pin only the transpiled text). These vectors are produced by
the reference's own listings (pkg/tests/fixtures/listing_nbody.c,
listing_diffusion.c), lowered by its transpiler's fallback backend and
compiled with g++ -O3 (oracle/build_ref.py -> oracle/_ref/libref_ieee_*.so).
Re-run after `make -C oracle` in a container that has /root/reference:

    python tests/golden/make_golden.py
"""
from __future__ import annotations

import pathlib
import sys

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

import oracle  # noqa: E402
from paper_2411_18889_b200.nbody import plummer_numpy, uniform_numpy  # noqa: E402

HERE = pathlib.Path(__file__).resolve().parent
EPS = 2.0 ** -6

# (name, generator, n, seed)
NBODY_CASES = [
    ("plummer256", "plummer", 256, 1),
    ("uniform300", "uniform", 300, 2),     # ragged: not a multiple of any tile size
    ("plummer1", "plummer", 1, 3),         # single particle: self term only
    ("coincident5", "coincident", 5, 4),   # duplicated positions: r = 0 pairs, eps > 0
]

# (name, shape, steps, (dx, dy, dz, dt, kappa), seed)
DIFF_CASES = [
    ("cube16", (16, 16, 16), 3, (1 / 16, 1 / 16, 1 / 16, 0.1 / 16 ** 2, 1.0), 3),
    ("aniso_12x20x24", (12, 20, 24), 4, (0.1, 0.08, 0.05, 2e-4, 1.3), 5),
    ("ragged_7x5x9", (7, 5, 9), 2, (1.0, 1.0, 1.0, 0.05, 1.0), 6),      # nz % 4 != 0
    ("thin_1x3x8", (1, 3, 8), 2, (1.0, 1.0, 1.0, 0.1, 1.0), 8),         # nx = 1: both i-clamps
    ("line_2x1x40", (2, 1, 40), 3, (1.0, 1.0, 1.0, 0.1, 1.0), 9),       # ny = 1
]


def particles(kind: str, n: int, seed: int) -> np.ndarray:
    if kind == "plummer":
        return plummer_numpy(n, seed)[0]
    if kind == "uniform":
        return uniform_numpy(n, seed)[0]
    if kind == "coincident":
        p = uniform_numpy(n, seed)[0]
        p[1] = p[0]
        p[3, :3] = p[2, :3]
        return p
    raise ValueError(kind)


def main() -> None:
    ref = oracle.Reference("ieee")
    out = {}
    for name, kind, n, seed in NBODY_CASES:
        pos = particles(kind, n, seed)
        out[f"nbody/{name}/pos"] = pos
        out[f"nbody/{name}/eps"] = np.float32(EPS)
        out[f"nbody/{name}/acc"] = ref.calc_acc(pos, pos, EPS, potential=False)
        out[f"nbody/{name}/acc_pot"] = ref.calc_acc(pos, pos, EPS, potential=True)
    # i-subset against a larger j-set (Ni != Nj, as in the sharded path)
    pos = plummer_numpy(1000, 11)[0]
    out["nbody/subset/ipos"] = pos[123:223].copy()
    out["nbody/subset/jpos"] = pos
    out["nbody/subset/eps"] = np.float32(EPS)
    out["nbody/subset/acc"] = ref.calc_acc(pos[123:223], pos, EPS)
    for name, shape, steps, params, seed in DIFF_CASES:
        f0 = np.random.default_rng(seed).random(shape, dtype=np.float32)
        out[f"diff/{name}/f0"] = f0
        out[f"diff/{name}/params"] = np.array(params, np.float32)
        out[f"diff/{name}/steps"] = np.int32(steps)
        out[f"diff/{name}/f"] = ref.diffusion_run(f0, steps, *params)
    np.savez_compressed(HERE / "golden.npz", **out)
    print(f"wrote {HERE / 'golden.npz'} ({len(out)} arrays)")


if __name__ == "__main__":
    main()
