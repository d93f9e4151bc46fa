mkdir -p gpurun_out
for b in trace_small trace_small_ldg trace_small trace_small_ldg; do echo "== $b"; ./scripts/$b 4096 40; ./scripts/$b 8192 40; done > gpurun_out/trace_small.log 2>&1
