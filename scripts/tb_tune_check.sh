# The two-step run's tuned plan at 512^3 / 1024^3 (verbose plan timing) and its effective GLUPS,
# repeated in fresh processes: how stable is the tuner's pick?
for rep in 1 2 3; do for g in ${GRIDS:-512 1024}; do SOLOMON_DIFF_TB_VERBOSE=1 timeout 300 python -c "
import sys; sys.path.insert(0,'.')
import torch, statistics, paper_2411_18889_b200 as b2
g=$g; f = b2.init_grid(g,g,g); sim = b2.Diffusion3D(f, 1/g,1/g,1/g, 0.1/g**2); sim.run(4); torch.cuda.synchronize()
ts=[]
for _ in range(3):
    e0,e1=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True); e0.record(); sim.run(20); e1.record(); torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1)/20)
print('tuned g',g,'GLUPS',round(g**3/statistics.median(ts)/1e6,1), flush=True)
" 2>&1 | grep -v score; done; done
