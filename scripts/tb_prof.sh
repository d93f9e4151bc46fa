ncu --set full --clock-control none --import-source on -k regex:k_diffusion_march2 -s 2 -c 1 -o gpurun_out/prof_tb python -c "
import sys; sys.path.insert(0,'.')
import torch, paper_2411_18889_b200 as b2
g=512; f = b2.init_grid(g,g,g); sim = b2.Diffusion3D(f, 1/g,1/g,1/g, 0.1/g**2); sim.run(8); torch.cuda.synchronize()
" > gpurun_out/prof_tb.log 2>&1
tail -3 gpurun_out/prof_tb.log
