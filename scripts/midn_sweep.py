"""Force-kernel variant sweep at mid N (tuning helper): SOLOMON_NBODY_VARIANT x SOLOMON_NBODY_WANT."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2411_18889_b200 as b2

for n in (8192, 16384, 32768, 65536):
    pos, _ = b2.plummer(n, 42)
    out = torch.empty_like(pos)
    for _ in range(3):
        b2.calc_acc(n, pos, out, n, pos, 2.0 ** -6)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    reps = 20
    ev[0].record()
    for _ in range(reps):
        b2.calc_acc(n, pos, out, n, pos, 2.0 ** -6)
    ev[1].record()
    torch.cuda.synchronize()
    ms = ev[0].elapsed_time(ev[1]) / reps
    print(json.dumps({"n": n, "variant": os.environ.get("SOLOMON_NBODY_VARIANT", "0"),
                      "want": os.environ.get("SOLOMON_NBODY_WANT", "4"), "us": ms * 1e3,
                      "ginter": n * n / (ms * 1e-3) / 1e9}), flush=True)
