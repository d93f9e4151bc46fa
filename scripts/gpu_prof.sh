# the round's ncu evidence (profile_round.sh) + a quick check of the parity-config timings
mkdir -p gpurun_out
TAG=${TAG:-r02} bash scripts/profile_round.sh
timeout 300 python scripts/small_configs.py --reps 5 > gpurun_out/small_configs_${TAG:-r02}.log 2>&1
