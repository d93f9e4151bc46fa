#!/bin/bash
# ncu evidence for a round (B200_PROFILING.md recipe): the launch list of a short bench run and
# one `--set full` capture per hot kernel, exported as raw CSV into gpurun_out/.
TAG=${TAG:-r02}
K=${KERNELS:-"force:k_force_fast march:k_diffusion_march tb2:k_diffusion_tb2 small:k_leapfrog_small resident:k_diffusion_resident"}
export PYTHONPATH=$PWD
mkdir -p gpurun_out
if [ -z "$NO_LAUNCHES" ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --dsteps 4 > gpurun_out/launches_bench_$TAG.log 2>&1
fi
for kv in $K; do
  w=${kv%%:*}; k=${kv#*:}
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 -f \
    -o gpurun_out/prof_${w}_$TAG python scripts/prof_workload.py $w > gpurun_out/prof_${w}_$TAG.log 2>&1
  ncu -i gpurun_out/prof_${w}_$TAG.ncu-rep --page raw --csv > gpurun_out/prof_${w}_${TAG}_raw.csv 2>/dev/null
  rm -f gpurun_out/prof_${w}_$TAG.ncu-rep
done
