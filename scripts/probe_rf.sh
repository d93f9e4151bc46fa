python - <<'PY'
import ctypes
p = ctypes.CDLL("paper_2411_18889_b200/lib/libsolomon_probe.so")
p.solomon_probe_pattern_tflops.restype = ctypes.c_double
p.solomon_probe_fp32_tflops.restype = ctypes.c_double
pk = p.solomon_probe_fp32_tflops(3)
print("ffma2 peak (2 flop/lane)", round(pk, 2))
names = ["ffma2 x,y,acc 3 pairs", "ffma2 x,y0(reuse),acc", "ffma x,y,acc scalar", "ffma2 x,x,acc",
         "fadd2 acc,x (2 pairs)", "fmul2 acc,x (2 pairs)", "ffma2 acc,s(.F32),x", "fadd2 acc,s(.F32)",
         "fmul2 acc,s(.F32)", "ffma2 acc,s,s"]
for m, n in enumerate(names):
    t = p.solomon_probe_pattern_tflops(m)
    flop = 1 if m in (4, 5, 7, 8) else 2
    print(f"{n:28s} {t:7.2f} T{'FLOP' if flop == 2 else 'op'}/s  -> instr rate {t / (pk / (1 if m != 2 else 1)) * (2 / flop) * (1 if m != 2 else 1):.3f} of FFMA2 peak")
PY
