mkdir -p gpurun_out
for tool in memcheck racecheck synccheck initcheck; do
  echo "== $tool"
  SOLOMON_DIFF_DIRECT_MAXCELLS=1000 timeout 900 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_workload.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "rc=$?"; tail -4 gpurun_out/sanitize_$tool.log
done
SOLOMON_DIFF_RESIDENT=0 SOLOMON_DIFF_DIRECT_MAXCELLS=0 timeout 600 compute-sanitizer --tool racecheck python -c "
import sys; sys.path.insert(0,'.')
import torch, paper_2411_18889_b200 as b2
f=torch.rand((24,40,128),device='cuda'); b2.Diffusion3D(f,0.1,0.1,0.1,1e-3,1.0).run(4)
f=torch.rand((12,9,1024),device='cuda'); b2.Diffusion3D(f,0.1,0.1,0.1,1e-3,1.0).run(2)  # 4-row tiles on 1024-float rows
f=torch.rand((10,13,384),device='cuda'); b2.Diffusion3D(f,0.1,0.1,0.1,1e-3,1.0).run(2)   # idle warps: 384-float rows
f=torch.rand((10,7,768),device='cuda'); b2.Diffusion3D(f,0.1,0.1,0.1,1e-3,1.0).run(2)    # idle warps: 768-float rows
torch.cuda.synchronize(); print('tb ok')" > gpurun_out/sanitize_tb.log 2>&1; echo "tb rc=$?"; tail -3 gpurun_out/sanitize_tb.log
for tool in memcheck racecheck; do
  timeout 900 compute-sanitizer --tool $tool --target-processes all --print-limit 20 python scripts/sanitize_halo.py > gpurun_out/sanitize_halo_$tool.log 2>&1
  echo "halo $tool rc=$?"; tail -3 gpurun_out/sanitize_halo_$tool.log
done
