"""Long-run physics checks of the leapfrog integrator on the GPU (the north star's KDK has no
reference counterpart; SURVEY.md §8f row 3 asks for energy / momentum diagnostics).

    python scripts/physics_check.py [--n N] [--steps S] [--out FILE]

* energy: relative drift of E = K + W over S KDK steps (Plummer, standard units, E0 = -1/4);
* momentum: |sum m v| stays at FP32 round-off of the initial (centre-of-mass frame) value;
* reversibility: S/2 steps forward, velocities negated, S/2 steps back -> the initial
  positions again up to FP32 round-off (leapfrog is time-symmetric);
* diffusion: a clamped-boundary eigenmode decays by the exact per-step factor, and the
  zero-flux ends conserve the mean (256^3, 1000 steps through Diffusion3D.run).
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2411_18889_b200 as b2  # noqa: E402


def total_energy(pos, vel, eps):
    out = torch.empty_like(pos)
    b2.calc_acc(pos.shape[0], pos, out, pos.shape[0], pos, eps, potential=True)
    ke, pe = b2.energy(pos, vel, out, eps)
    return ke + pe


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1 << 16)
    ap.add_argument("--steps", type=int, default=2048)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    eps, dt = 2.0 ** -6, 2.0 ** -7
    pos, vel = b2.plummer(args.n, 42)
    e0 = total_energy(pos, vel, eps)
    p0 = (pos[:, 3:4].double() * vel[:, :3].double()).sum(0)
    lf = b2.Leapfrog(pos.clone(), vel.clone(), eps, dt)
    rows = []
    done = 0
    for chunk in (args.steps // 4,) * 4:
        lf.step(chunk)
        done += chunk
        e = total_energy(lf.pos, lf.vel, eps)
        p = (lf.pos[:, 3:4].double() * lf.vel[:, :3].double()).sum(0)
        rows.append({"steps": done, "time": done * dt, "energy": e, "rel_drift": abs(e - e0) / abs(e0),
                     "momentum": float(p.norm()), "momentum_0": float(p0.norm())})
        print(json.dumps(rows[-1]), flush=True)
    # reversibility
    half = args.steps // 2
    fw = b2.Leapfrog(pos.clone(), vel.clone(), eps, dt)
    fw.step(half)
    fw.vel[:, :3].neg_()
    back = b2.Leapfrog(fw.pos.clone(), fw.vel.clone(), eps, dt)
    back.step(half)
    err = float(((back.pos[:, :3] - pos[:, :3]).norm() / pos[:, :3].norm()).item())
    rows.append({"reversibility_relL2_pos": err, "steps_each_way": half})
    print(json.dumps(rows[-1]), flush=True)
    # diffusion: a clamped-boundary eigenmode decays by an exact factor per step
    # (f = 1 + a cos(pi (i + 1/2) / nx) is an eigenvector of the listing's clamped stencil:
    # lambda = 1 - 2 ce (1 - cos(pi / nx))), and the clamped (zero-flux) ends conserve the mean
    g, dsteps = 256, 1000
    dx = 1.0 / g
    dargs = (dx, dx, dx, 0.1 * dx * dx, 1.0)
    i = torch.arange(g, dtype=torch.float64, device="cuda")
    mode = torch.cos(torch.pi * (i + 0.5) / g)
    f0 = (1.0 + 0.5 * mode)[:, None, None].expand(g, g, g).contiguous()
    sim = b2.Diffusion3D(f0.float(), *dargs)
    sim.run(dsteps)
    ce = 1.0 * dargs[3] / (dx * dx)
    lam = 1.0 - 2.0 * ce * (1.0 - torch.cos(torch.tensor(torch.pi / g, dtype=torch.float64)))
    want = 1.0 + 0.5 * lam ** dsteps * mode
    got = sim.field.double().mean(dim=(1, 2))
    rows.append({"diffusion_grid": g, "steps": dsteps, "decay_factor": float(lam ** dsteps),
                 "mode_relL2": float(((got - want).norm() / (want - 1.0).norm()).item()),
                 "mean_drift": float(abs(sim.field.double().mean().item() - 1.0))})
    print(json.dumps(rows[-1]), flush=True)
    if args.out:
        with open(args.out, "w") as fh:
            for r in rows:
                fh.write(json.dumps(r) + "\n")


if __name__ == "__main__":
    main()
