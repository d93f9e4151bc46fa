"""One hot kernel, launched a few times, for `ncu --set full -k regex:<kernel> -s 1 -c 1`.

    python scripts/prof_workload.py force|march|tb2|small|resident
"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2411_18889_b200 as b2  # noqa: E402

what = sys.argv[1]
EPS, DT = 2.0 ** -6, 2.0 ** -7
if what == "force":  # k_force_fast, N = 2^20 (configs[2]), in-kernel chunk reduction
    pos, _ = b2.plummer(1 << 20, 42)
    acc = torch.empty_like(pos)
    ws = b2.workspace(1 << 20, 1 << 20)
    for _ in range(2):
        b2.calc_acc(1 << 20, pos, acc, 1 << 20, pos, EPS, ws=ws)
elif what in ("march", "tb2"):  # 512^3 single step / two steps per pass
    g = 512
    sim = b2.Diffusion3D(b2.init_grid(g, g, g), 1 / g, 1 / g, 1 / g, 0.1 / g ** 2)
    for _ in range(3):
        if what == "march":
            b2.diffusion3d(g, g, g, 1 / g, 1 / g, 1 / g, 0.1 / g ** 2, 1.0, sim.f, sim._fn)
        else:
            sim.run(2)
elif what == "small":  # configs[0]: N = 4096, 16 KDK steps in one launch
    pos, vel = b2.plummer(4096, 42)
    for _ in range(3):
        lf = b2.Leapfrog(pos.clone(), vel.clone(), EPS, DT)
        lf.step(16)
elif what == "resident":  # configs[1]: 128^3, 100 steps in one launch
    g = 128
    for _ in range(3):
        sim = b2.Diffusion3D(b2.init_grid(g, g, g), 1 / g, 1 / g, 1 / g, 0.1 / g ** 2)
        sim.run(100)
torch.cuda.synchronize()
