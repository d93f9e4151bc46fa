"""e2e of the diffusion3d drop-in on pinned host buffers (tuning helper for the chunked pipeline)."""
import ctypes, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2411_18889_b200 as b2

lib = b2.load()
g = int(sys.argv[1]) if len(sys.argv) > 1 else 512
f = b2.init_grid(g, g, g, seed=7).cpu().pin_memory()
fn = torch.empty_like(f).pin_memory()
d = 1.0 / g
P = ctypes.c_void_p
for _ in range(2):
    lib.diffusion3d(g, g, g, d, d, d, 0.1 * d * d, 1.0, P(f.data_ptr()), P(fn.data_ptr()))
t0 = time.perf_counter()
for _ in range(5):
    lib.diffusion3d(g, g, g, d, d, d, 0.1 * d * d, 1.0, P(f.data_ptr()), P(fn.data_ptr()))
t = (time.perf_counter() - t0) / 5
print(f"g={g} e2e {t*1e3:.2f} ms  {g**3/t/1e9:.2f} GLUPS")
