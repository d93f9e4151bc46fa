"""Long-run physics checks of the leapfrog integrator on the GPU (the north star's KDK has no
reference counterpart; SURVEY.md §8f row 3 asks for energy / momentum diagnostics).

    python scripts/physics_check.py [--n N] [--steps S] [--out FILE]

* energy: relative drift of E = K + W over S KDK steps (Plummer, standard units, E0 = -1/4);
* momentum: |sum m v| stays at FP32 round-off of the initial (centre-of-mass frame) value;
* reversibility: S/2 steps forward, velocities negated, S/2 steps back -> the initial
  positions again up to FP32 round-off (leapfrog is time-symmetric).
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
    if args.out:
        with open(args.out, "w") as fh:
            for r in rows:
                fh.write(json.dumps(r) + "\n")


if __name__ == "__main__":
    main()
