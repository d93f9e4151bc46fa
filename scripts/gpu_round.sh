# Round evidence: GPU tests, smoke, bench (both arms), ncu launch list, ncu --set full of the two hot kernels.
set -x
TAG=${TAG:-r01}
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q 2>&1 | tail -5
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; tail -3 gpurun_out/bench_$TAG.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_$TAG.json 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-configs --dsteps 10 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_force_fast -s 2 -c 1 -o gpurun_out/prof_force_$TAG python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-diffusion --no-configs > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_diffusion_march -s 5 -c 1 -o gpurun_out/prof_diff_$TAG python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-configs --dsteps 2 --particles 65536 > /dev/null 2>&1
ls -la gpurun_out
