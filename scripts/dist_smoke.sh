python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --dist --steps 2 --warmup 1 --no-cpu-baseline --no-configs > gpurun_out/dist.log 2>&1
grep -v "^\s*$" gpurun_out/dist.log | grep -iE "error|Traceback|File|line" | head -30
