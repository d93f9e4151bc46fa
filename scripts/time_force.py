"""Tuning helper: time k_force_fast variants (SOLOMON_NBODY_VARIANT) at N=2^20 on one GPU.

    python scripts/time_force.py 0 11 12 ...      # one subprocess per variant

Prints ms per force evaluation, Ginteractions/s, the fraction of the live FP32
peak, and the relL2 of a sampled slice against the oracle restatement.
"""
import ctypes
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def one(n: int) -> None:
    import numpy as np
    import torch

    import oracle
    import paper_2411_18889_b200 as b2
    from paper_2411_18889_b200 import _lib

    lib = b2.load()
    probe = ctypes.CDLL(os.path.join(ROOT, "paper_2411_18889_b200", "lib", "libsolomon_probe.so"))
    probe.solomon_probe_fp32_tflops.restype = ctypes.c_double
    peak = probe.solomon_probe_fp32_tflops(3)
    pos_np, _ = b2.plummer_numpy(n, 42)
    pos = torch.from_numpy(pos_np).cuda()
    nch = lib.b2_calc_acc_nchunks(n, 0)
    part = torch.empty((nch * n, 4), dtype=torch.float32, device="cuda")
    acc = torch.empty_like(pos)
    sh = _lib.stream_handle(pos.device)

    def force():
        _lib.check(lib.b2_calc_acc_partials(n, pos.data_ptr(), n, pos.data_ptr(), 2.0 ** -6, 0, part.data_ptr(), sh),
                   "partials")

    force()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record()
    for _ in range(3):
        force()
    ev[1].record()
    torch.cuda.synchronize()
    ms = ev[0].elapsed_time(ev[1]) / 3
    _lib.check(lib.b2_kdk_update(n, None, None, acc.data_ptr(), part.data_ptr(), nch, 0.0, 0.0, 0.0,
                                 _lib.B2_KDK_REDUCE, sh), "reduce")
    idx = np.random.default_rng(0).choice(n, 256, replace=False)
    want = oracle.Restatement().calc_acc(pos_np[idx], pos_np, 2.0 ** -6)
    got = acc.cpu().numpy()[idx]
    err = np.linalg.norm(got[:, :3] - want[:, :3]) / np.linalg.norm(want[:, :3])
    tf = 20.0 * n * n / (ms * 1e-3) / 1e12
    print(f"variant {os.environ.get('SOLOMON_NBODY_VARIANT', '0'):>3}  {ms:8.2f} ms  "
          f"{n * n / (ms * 1e-3) / 1e9:8.1f} Ginter/s  {tf:6.2f} TF  frac {tf / peak:.4f}  relL2 {err:.2e}", flush=True)


if __name__ == "__main__":
    n = int(os.environ.get("N", 1 << 20))
    if os.environ.get("_ONE"):
        one(n)
    else:
        for v in sys.argv[1:] or ["0"]:
            env = dict(os.environ, SOLOMON_NBODY_VARIANT=v, _ONE="1")
            subprocess.run([sys.executable, __file__], env=env, check=False)
