# A/B of a compile-time k_diffusion_tb2 variant: $FLAG builds vs the default, effective GLUPS
# (three interleaved repeats) + the temporal-blocking bit-identity tests on the variant.
FLAG=${FLAG:--DB2_TB_SHFL2=1}
cp paper_2411_18889_b200/lib/libsolomon_b200.so /tmp/lib_default.so
SOLOMON_NVCC_EXTRA="$FLAG" python -c "from paper_2411_18889_b200 import build as b; b.build(force=True)" && cp paper_2411_18889_b200/lib/libsolomon_b200.so /tmp/lib_variant.so
SOLOMON_DIFF_DIRECT_MAXCELLS=0 timeout 600 python -m pytest tests/test_parity_gpu.py -x -q -k "temporal or two_steps or run2_planes or bit_identical" -p no:cacheprovider 2>&1 | tail -2
for rep in 1 2 3; do for v in default variant; do cp /tmp/lib_$v.so paper_2411_18889_b200/lib/libsolomon_b200.so; for g in ${GRIDS:-512 1024}; do timeout 300 python -c "
import sys; sys.path.insert(0,'.')
import torch, paper_2411_18889_b200 as b2
g=$g; f = b2.init_grid(g,g,g); sim = b2.Diffusion3D(f, 1/g,1/g,1/g, 0.1/g**2); sim.run(4); torch.cuda.synchronize()
n = 40 if g < 1024 else 10
e0,e1=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True); e0.record(); sim.run(n); e1.record(); torch.cuda.synchronize()
ms=e0.elapsed_time(e1)/n; print('$v g',g,'GLUPS (effective)',round(g**3/ms/1e6,1))
"; done; done; done
cp /tmp/lib_default.so paper_2411_18889_b200/lib/libsolomon_b200.so
