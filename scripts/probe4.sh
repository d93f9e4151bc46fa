python - <<'PY'
import ctypes
p = ctypes.CDLL("paper_2411_18889_b200/lib/libsolomon_probe.so")
p.solomon_probe_nbody_inner.restype = ctypes.c_double
p.solomon_probe_fp32_tflops.restype = ctypes.c_double
print("ffma2 peak", p.solomon_probe_fp32_tflops(3))
for s, name in ((0, "constant/UR j"), (1, "shared dup j")):
    for _ in range(2):
        print(name, round(p.solomon_probe_nbody_inner(s), 2), "TF(20-flop)")
PY
