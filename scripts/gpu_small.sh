mkdir -p gpurun_out
timeout 300 python scripts/midn_sweep.py > gpurun_out/midn.log 2>&1
timeout 600 python scripts/leapfrog_sizes.py > gpurun_out/lf_sizes.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gputest_small.log 2>&1
echo rc=$? >> gpurun_out/gputest_small.log
