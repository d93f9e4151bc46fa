"""Accuracy of the active force variant (SOLOMON_NBODY_VARIANT) vs the oracle (tuning helper)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle, paper_2411_18889_b200 as b2
o = oracle.Restatement()
for n in (8192, 65536):
    pos, _ = b2.plummer_numpy(n, 42)
    idx = np.random.default_rng(0).choice(n, 1024, replace=False)
    want = o.calc_acc(pos[idx], pos, 2.0 ** -6, potential=True)
    got = b2.accelerations(torch.from_numpy(pos).cuda(), 2.0 ** -6, potential=True).cpu().numpy()[idx]
    e = np.linalg.norm(got[:, :3] - want[:, :3]) / np.linalg.norm(want[:, :3])
    ep = np.linalg.norm(got[:, 3] - want[:, 3]) / np.linalg.norm(want[:, 3])
    print(f"  variant {os.environ.get('SOLOMON_NBODY_VARIANT','0')} n={n} relL2 acc {e:.2e} pot {ep:.2e}")
