"""Small workload touching every kernel, for compute-sanitizer (memcheck/racecheck/synccheck)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2411_18889_b200 as b2

dev = "cuda"
pos, vel = b2.plummer(3000, 1)                         # ragged N: small variant, chunk padding
for pot in (False, True):
    b2.accelerations(pos, 2 ** -6, potential=pot)
    b2.accelerations(pos[:1000].contiguous(), 2 ** -6, pos, potential=pot, exact=True)
big, _ = b2.plummer(40000, 2)
b2.accelerations(big[:20000].contiguous(), 2 ** -6, big)     # large variant path
lf = b2.Leapfrog(pos.clone(), vel.clone(), 2 ** -6, 2 ** -7); lf.step(3)
huge, _ = b2.plummer(70000, 3)
b2.accelerations(huge, 2 ** -6, huge[:4096].contiguous())   # Ni > 63488: in-kernel ring reduction
for n in (4096, 8192):                                      # persistent path: 2 and 4 pair groups
    p2, v2 = b2.plummer(n, 4)
    b2.Leapfrog(p2, v2, 2 ** -6, 2 ** -7, potential=n == 8192).step(2)
for shape in [(20, 24, 128), (7, 5, 9), (5, 3, 512), (3, 4, 100)]:
    f = torch.rand(shape, device=dev); fn = torch.empty_like(f)
    b2.diffusion3d(*shape, 0.1, 0.1, 0.1, 1e-3, 1.0, f, fn)
    b2.Diffusion3D(f.clone(), 0.1, 0.1, 0.1, 1e-3, 1.0).run(3)
f = torch.rand((40, 64, 512), device=dev)
b2.Diffusion3D(f.clone(), 0.1, 0.1, 0.1, 1e-3, 1.0).run(2)   # march kernel (> direct threshold? no) 
fl = f[:20].contiguous(); o = torch.empty_like(fl)
b2.diffusion3d_slab(fl, o, f[20].contiguous(), None, 0.1, 0.1, 0.1, 1e-3, 1.0)
h = np.random.default_rng(0).random((33, 20, 16), dtype=np.float32); hn = np.empty_like(h)
lib = b2.load()
lib.diffusion3d(33, 20, 16, 0.1, 0.1, 0.1, 1e-3, 1.0, h.ctypes.data_as(ctypes.c_void_p), hn.ctypes.data_as(ctypes.c_void_p))
torch.cuda.synchronize()
print("workload ok")
