mkdir -p gpurun_out
for b in trace_small trace_small_ws0 trace_small trace_small_ws0; do echo "== $b"; ./scripts/$b 4096 40; done > gpurun_out/trace_small.log 2>&1
./scripts/trace_small 2048 40 >> gpurun_out/trace_small.log 2>&1
./scripts/trace_small 4736 40 >> gpurun_out/trace_small.log 2>&1
timeout 300 python scripts/small_configs.py --reps 5 --which 0 > gpurun_out/small0.log 2>&1
timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "leapfrog or small or persistent or chunk or fault" > gpurun_out/gputest_small.log 2>&1
echo rc=$? >> gpurun_out/gputest_small.log
