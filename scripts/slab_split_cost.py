"""Cost of the overlapped SlabDiffusion.run pass on one GPU without an exchange: one
two-step pass over a halo-extended 1024^3/8 slab (2 + 128 + 2 planes) as one launch, vs the
interior (b2_diffusion3d_run2_planes) + the launch of both 2-plane edges the overlap issues."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2411_18889_b200 as b2  # noqa: E402
from paper_2411_18889_b200.distributed import CudaSlabKernels  # noqa: E402

g = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
nxl = g // 8
args = (1 / g, 1 / g, 1 / g, 0.1 / g ** 2, 1.0)
f = torch.rand((nxl + 4, g, g), device="cuda")
fn = torch.empty_like(f)
k = CudaSlabKernels(*args)
b2.diffusion.plan(f, fn, *args, nsteps=2)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]


def timeit(fn_, reps=20):
    for _ in range(3):
        fn_()
    torch.cuda.synchronize()
    ev[0].record()
    for _ in range(reps):
        fn_()
    ev[1].record()
    torch.cuda.synchronize()
    return ev[0].elapsed_time(ev[1]) / reps * 1e3


whole = timeit(lambda: k.run2(f, fn))
lo_h = 2


def split():
    k.run2_planes(f, fn, lo_h + 2, lo_h + nxl - 2)
    k.run2_planes(f, fn, lo_h, lo_h + 2, lo_h + nxl - 2, lo_h + nxl)


sp = timeit(split)
interior = timeit(lambda: k.run2_planes(f, fn, lo_h + 2, lo_h + nxl - 2))
print(f"slab {nxl}+4 planes of {g}^2: whole pass {whole:.1f} us, interior {interior:.1f} us, "
      f"interior + 2 edges {sp:.1f} us (edges {sp - interior:.1f} us)")
