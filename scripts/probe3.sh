mkdir -p gpurun_out
python - <<'PY'
import ctypes
p = ctypes.CDLL("paper_2411_18889_b200/lib/libsolomon_probe.so")
p.solomon_probe_pattern_tflops.restype = ctypes.c_double
p.solomon_probe_fp32_tflops.restype = ctypes.c_double
print("ffma2 peak", p.solomon_probe_fp32_tflops(3))
for m, name in enumerate(["ffma2 3 distinct pairs", "ffma2 shared operand", "ffma scalar 3 distinct", "ffma2 2 distinct pairs"]):
    print(name, round(p.solomon_probe_pattern_tflops(m), 2))
PY
for nst in 2 3; do for sp in 4 8; do SOLOMON_DIFF_NST=$nst SOLOMON_DIFF_SPLITS=$sp python scripts/time_diffusion.py; done; done
SOLOMON_DIFF_NST=3 SOLOMON_DIFF_OCC=3 SOLOMON_DIFF_S=2 python scripts/time_diffusion.py
SOLOMON_DIFF_NST=2 SOLOMON_DIFF_OCC=3 SOLOMON_DIFF_S=2 python scripts/time_diffusion.py
SOLOMON_DIFF_NST=3 python scripts/time_diffusion.py 1024 20
SOLOMON_DIFF_NST=3 python scripts/time_diffusion.py 256 200
ncu --set full --clock-control none --import-source on -k regex:k_force_fast -s 2 -c 1 -o gpurun_out/prof_force_v0 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-diffusion > /dev/null 2>&1
ls gpurun_out
