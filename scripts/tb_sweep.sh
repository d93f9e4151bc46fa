# k_diffusion_tb2 plan sweep: tile height TJ x i-split count at one grid size ($G), effective GLUPS.
G=${G:-512}
for tj in ${TJS:-7 8 9 10}; do for sp in ${SPLITS:-1 2 3 4 5 6 8 10 12 14 16}; do
SOLOMON_DIFF_TB_VERBOSE=1 SOLOMON_DIFF_TB_TJ=$tj SOLOMON_DIFF_TB_SPLITS=$sp timeout 300 python -c "
import sys; sys.path.insert(0,'.')
import torch, paper_2411_18889_b200 as b2
g=$G; f = b2.init_grid(g,g,g); sim = b2.Diffusion3D(f, 1/g,1/g,1/g, 0.1/g**2); sim.run(4); torch.cuda.synchronize()
n = 40 if g < 1024 else 10
e0,e1=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True); e0.record(); sim.run(n); e1.record(); torch.cuda.synchronize()
ms=e0.elapsed_time(e1)/n; print('TJ=$tj splits=$sp g',g,'GLUPS',round(g**3/ms/1e6,1), flush=True)
" 2>&1 | sort -u | tr '\n' ' '; echo; done; done
