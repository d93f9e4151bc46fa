mkdir -p gpurun_out
for v in 0 4 5 6 7 8 9; do
  SOLOMON_NBODY_VARIANT=$v python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-diffusion \
    | python -c "import json,sys; d=json.load(sys.stdin); r=d['roofline']; print('variant $v', round(d['value'],1), 'Ginter/s frac', round(r['frac'],4), 'force_ms', round(r['force_ms'],2))"
done
python scripts/time_diffusion.py
SOLOMON_DIFF_NST=3 python scripts/time_diffusion.py
SOLOMON_DIFF_SPLITS=2 python scripts/time_diffusion.py
SOLOMON_DIFF_SPLITS=8 python scripts/time_diffusion.py
SOLOMON_DIFF_SPLITS=16 python scripts/time_diffusion.py
SOLOMON_DIFF_OCC=4 SOLOMON_DIFF_S=2 python scripts/time_diffusion.py
SOLOMON_DIFF_OCC=3 SOLOMON_DIFF_S=2 python scripts/time_diffusion.py
SOLOMON_DIFF_OCC=2 SOLOMON_DIFF_S=2 python scripts/time_diffusion.py
SOLOMON_DIFF_OCC=4 SOLOMON_DIFF_S=1 python scripts/time_diffusion.py
SOLOMON_DIFF_OCC=4 SOLOMON_DIFF_S=2 SOLOMON_DIFF_SPLITS=8 python scripts/time_diffusion.py
SOLOMON_DIFF_OCC=1 SOLOMON_DIFF_S=4 python scripts/time_diffusion.py
python scripts/time_diffusion.py 1024 20
python -c "
import torch,time
a=torch.empty(1<<28, dtype=torch.float32, device='cuda'); b=torch.empty_like(a)
for _ in range(3): b.copy_(a)
torch.cuda.synchronize(); e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20): b.copy_(a)
e1.record(); torch.cuda.synchronize(); ms=e0.elapsed_time(e1)/20
print('torch copy 1 GiB->1 GiB', ms, 'ms', 2*(1<<30)/ms/1e6, 'GB/s')
"
