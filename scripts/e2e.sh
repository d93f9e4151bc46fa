python -m pytest tests/test_parity_gpu.py -q -x -k "dropin" 2>&1 | tail -2
python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-configs --n 65536 | python -c "import json,sys; d=json.load(sys.stdin)['secondary']['diffusion']; print('diff e2e', d['e2e'], 'value', d['value'])"
