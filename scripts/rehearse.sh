#!/bin/bash
# Full-size rehearsal of the N>1 bench path on ONE B200: W ranks share cuda:0 (--same-device:
# gloo control plane, p2p transports, NCCL cannot put two ranks on one GPU). Not a scaling
# number -- it proves the N>1 line is produced (parity, e2e, anchor) at BASELINE sizes:
# configs[3] N = 2^22 i-shards, configs[4] 1024^3 i-slabs.
W=${1:-2}
TAG=${TAG:-r02}
shift
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $W --master-addr 127.0.0.1 \
  --master-port $((29600 + W)) bench.py --gpus $W --same-device --steps ${STEPS:-2} --warmup 3 "$@" \
  --detail gpurun_out/rehearse_w${W}_$TAG.json > gpurun_out/rehearse_w${W}_$TAG.out 2> gpurun_out/rehearse_w${W}_$TAG.err
echo "rehearse W=$W rc=$?" >> gpurun_out/rehearse_w${W}_$TAG.err
