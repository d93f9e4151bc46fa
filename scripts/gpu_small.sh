mkdir -p gpurun_out
timeout 600 python scripts/leapfrog_sizes.py 4096 4736 5120 6144 7168 8192 9472 12288 > gpurun_out/lf_sizes.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gputest_small.log 2>&1
echo rc=$? >> gpurun_out/gputest_small.log
