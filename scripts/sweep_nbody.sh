# Sweep the fast force-kernel launch variants (SOLOMON_NBODY_VARIANT) at N=2^20.
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for v in ${VARIANTS:-0 2 3 4 5 6 7 8 9}; do
  SOLOMON_NBODY_VARIANT=$v python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-diffusion \
    | python -c "import json,sys; d=json.load(sys.stdin); r=d['roofline']; print('variant $v', round(d['value'],1), 'Ginter/s frac', round(r['frac'],4), 'force_ms', round(r['force_ms'],2))"
done
python bench.py --steps 1 --warmup 1 --no-cpu-baseline --n 65536 --dsteps 100 | python -c "import json,sys; d=json.load(sys.stdin)['secondary']['diffusion']; print('diffusion', d['value'], d['roofline'])"
