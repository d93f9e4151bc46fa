for v in ${VARIANTS:-0 3 4 5 6 7 8 9}; do
  SOLOMON_NBODY_VARIANT=$v python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-diffusion \
    | python -c "import json,sys; d=json.load(sys.stdin); r=d['roofline']; print('variant $v', round(d['value'],1), 'Ginter/s frac', round(r['frac'],4), 'force_ms', round(r['force_ms'],2))"
  SOLOMON_NBODY_VARIANT=$v python scripts/check_variant.py
done
