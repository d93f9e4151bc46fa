mkdir -p gpurun_out
(python scripts/slab_split_cost.py 1024; python scripts/slab_split_cost.py 512) > gpurun_out/slab_split.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "run2_planes or p2p or distributed or slab or temporal or bit_identical" > gpurun_out/gputest_slab.log 2>&1
echo rc=$? >> gpurun_out/gputest_slab.log
