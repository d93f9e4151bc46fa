mkdir -p gpurun_out
for m in 64 128; do for w in 4 2; do echo "== midchunks $m want $w"; SOLOMON_NBODY_WANT=$w SOLOMON_NBODY_MIDCHUNKS=$m timeout 600 python scripts/leapfrog_sizes.py 12288 16384 24576 32768; done; done > gpurun_out/lf_mid.log 2>&1
