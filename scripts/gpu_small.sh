mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_distributed_gpu.py -m gpu -x -q -p no:cacheprovider -k "nvls or p2p_fused_allgather or match_single" > gpurun_out/gputest_nvls.log 2>&1
echo rc=$? >> gpurun_out/gputest_nvls.log
