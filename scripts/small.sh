python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for m in 0 1; do SOLOMON_DIFF_MULTI=$m python -c "
import sys; sys.path.insert(0,'.')
import torch, paper_2411_18889_b200 as b2
for g in (64,128,256):
  f = b2.init_grid(g,g,g); sim = b2.Diffusion3D(f, 1/g,1/g,1/g, 0.1/g**2); sim.run(10); torch.cuda.synchronize()
  e0,e1=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True); e0.record(); sim.run(100); e1.record(); torch.cuda.synchronize()
  ms=e0.elapsed_time(e1)/100; print('multi=$m g',g,'us/step',round(ms*1e3,2),'GLUPS',round(g**3/ms/1e6,1))
"; done
python scripts/time_diffusion.py 128 200
python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-diffusion --n 65536 | python -c "import json,sys; d=json.load(sys.stdin)['parity_configs']; print({k:(v['gpu_ms'],v.get('parity',v.get('parity_relL2'))) for k,v in d.items()})"
