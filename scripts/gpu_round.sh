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
# k_diffusion_march at 512^3: the first launches time candidate plans (first step of the shape); launch 45 is a timed step
ncu --set full --clock-control none --import-source on -k regex:k_diffusion_march -s 45 -c 1 -o gpurun_out/prof_diff_$TAG python scripts/time_diffusion.py 512 50 > /dev/null 2>&1
# k_diffusion_tb2: launches 0-11 time the four candidate plans (first run of the shape), 12-13 are the chosen plan
SOLOMON_DIFF_TEMPORAL=1 ncu --set full --clock-control none --import-source on -k regex:k_diffusion_tb2 -s 13 -c 1 -o gpurun_out/prof_tb2_$TAG python -c "
import sys; sys.path.insert(0,'.')
import torch, paper_2411_18889_b200 as b2
g=512; sim = b2.Diffusion3D(b2.init_grid(g,g,g), 1/g,1/g,1/g, 0.1/g**2); sim.run(4); torch.cuda.synchronize()  # launches 0-11 time 4 candidate plans, 12-13 the chosen one" > /dev/null 2>&1
# the persistent small-problem paths (BASELINE configs[0] / [1])
ncu --set full --clock-control none --import-source on -k regex:k_leapfrog_small -s 3 -c 1 -o gpurun_out/prof_small_$TAG python scripts/small_configs.py --which 0 --reps 3 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_diffusion_resident -s 2 -c 1 -o gpurun_out/prof_res_$TAG python scripts/small_configs.py --which 1 --reps 3 > /dev/null 2>&1
ls -la gpurun_out
