# Interleaved A/B of k_diffusion_tb2 i-split counts at one grid ($G, splits $VALS): is the tuner's pick real?
G=${G:-1024}
for rep in 1 2 3; do for sp in ${VALS:-4 8}; do SOLOMON_DIFF_TB_TJ=${TJ:-4} SOLOMON_DIFF_TB_SPLITS=$sp timeout 300 python -c "
import sys; sys.path.insert(0,'.')
import torch, paper_2411_18889_b200 as b2
g=$G; f = b2.init_grid(g,g,g); sim = b2.Diffusion3D(f, 1/g,1/g,1/g, 0.1/g**2); sim.run(4); torch.cuda.synchronize()
n = 20
e0,e1=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True); e0.record(); sim.run(n); e1.record(); torch.cuda.synchronize()
ms=e0.elapsed_time(e1)/n; print('splits=$sp g',g,'GLUPS',round(g**3/ms/1e6,1), flush=True)
"; done; done
