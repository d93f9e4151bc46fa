"""Time b2_diffusion3d at g^3 back to back (tuning helper; env knobs SOLOMON_DIFF_*)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2411_18889_b200 as b2

g = int(sys.argv[1]) if len(sys.argv) > 1 else 512
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 100
f = b2.init_grid(g, g, g, seed=7)
fn = torch.empty_like(f)
dx = 1.0 / g
args = (dx, dx, dx, 0.1 * dx * dx, 1.0)
for i in range(5):
    b2.diffusion3d(g, g, g, *args, f, fn); f, fn = fn, f
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for i in range(steps):
    b2.diffusion3d(g, g, g, *args, f, fn); f, fn = fn, f
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / steps
knobs = {k: v for k, v in os.environ.items() if k.startswith("SOLOMON_DIFF")}
print(json.dumps({"g": g, "ms": round(ms, 4), "glups": round(g**3 / ms / 1e6, 1), "gbs": round(8 * g**3 / ms / 1e6, 1), **knobs}))
