# A/B of a k_diffusion_tb2 variant knob ($KNOB over $VALS, interleaved): bit-identity tests with $KNOB=$TESTVAL, then effective GLUPS.
KNOB=${KNOB:-SOLOMON_DIFF_TB_SHFL}
env $KNOB=${TESTVAL:-1} SOLOMON_DIFF_DIRECT_MAXCELLS=0 timeout 600 python -m pytest tests/test_parity_gpu.py tests/test_properties_gpu.py -x -q -k "temporal or two_steps or config1 or bit_identical" 2>&1 | tail -2
for rep in 1 2 3; do for g in ${GRIDS:-256 512 1024}; do for v in ${VALS:-1 0}; do env $KNOB=$v timeout 300 python -c "
import sys; sys.path.insert(0,'.')
import torch, paper_2411_18889_b200 as b2
g=$g; f = b2.init_grid(g,g,g); sim = b2.Diffusion3D(f, 1/g,1/g,1/g, 0.1/g**2); sim.run(4); torch.cuda.synchronize()
n = 40 if g < 1024 else 10
e0,e1=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True); e0.record(); sim.run(n); e1.record(); torch.cuda.synchronize()
ms=e0.elapsed_time(e1)/n; print('$KNOB=$v g',g,'us/step',round(ms*1e3,2),'GLUPS (effective)',round(g**3/ms/1e6,1))
"; done; done; done
