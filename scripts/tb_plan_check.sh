# k_diffusion_tb2 at one grid: the tuned plan (verbose) and then forced tile heights x splits.
G=${G:-1024}
for rep in 1 2; do SOLOMON_DIFF_TB_VERBOSE=1 timeout 300 python -c "
import sys; sys.path.insert(0,'.')
import torch, paper_2411_18889_b200 as b2
g=$G; f = b2.init_grid(g,g,g); sim = b2.Diffusion3D(f, 1/g,1/g,1/g, 0.1/g**2); sim.run(4); torch.cuda.synchronize()
n = 20
e0,e1=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True); e0.record(); sim.run(n); e1.record(); torch.cuda.synchronize()
ms=e0.elapsed_time(e1)/n; print('tuned g',g,'GLUPS',round(g**3/ms/1e6,1), flush=True)
" 2>&1; done
TJS=${TJS:-3 4} SPLITS=${SPLITS:-1 2 4 7 8} G=$G bash scripts/tb_sweep.sh
