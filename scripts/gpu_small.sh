mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_faults_gpu.py tests/test_parity_gpu.py -m gpu -x -q -p no:cacheprovider -k "fault or expired or leapfrog or persistent" > gpurun_out/gputest_faults.log 2>&1
echo rc=$? >> gpurun_out/gputest_faults.log
