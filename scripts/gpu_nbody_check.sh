# n-body change check: the bit-identity / parity GPU tests of the n-body paths, the phase
# trace of the persistent small-N leapfrog, and Leapfrog.step(16) across N.
mkdir -p gpurun_out
TAG=${TAG:-x}
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "leapfrog or fused or chunk or nbody or calc_acc or kdk or shard or small" > gpurun_out/nb_tests_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/nb_tests_$TAG.log
./scripts/trace_small 4096 40 > gpurun_out/trace_small_$TAG.log 2>&1
./scripts/trace_small 8192 40 >> gpurun_out/trace_small_$TAG.log 2>&1
timeout 600 python scripts/leapfrog_sizes.py 4096 8192 16384 32768 > gpurun_out/lf_sizes_$TAG.log 2>&1
