#!/bin/bash
# One GPU session: tests, smoke, the N=1 bench (compact line + full record), and a world-2
# same-device rehearsal of the N>1 bench path. Outputs land in gpurun_out/.
set -x
TAG=${TAG:-r02}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gputest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest_$TAG.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1
[ -n "$AB" ] && timeout 300 python scripts/ab_force.py > gpurun_out/ab_force_$TAG.log 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 --detail gpurun_out/bench_detail_$TAG.json > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
echo "bench rc=$?" >> gpurun_out/bench_$TAG.err
