ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_small.csv python -c "
import sys; sys.path.insert(0,'.')
import torch, paper_2411_18889_b200 as b2
pos, vel = b2.plummer(4096, 42)
lf = b2.Leapfrog(pos, vel, 2**-6, 2**-7); lf.step(4)
f = b2.init_grid(128,128,128); sim = b2.Diffusion3D(f, 1/128,1/128,1/128, 0.1/128**2); sim.run(4)
torch.cuda.synchronize()
" > /dev/null 2>&1
grep -v "^==" gpurun_out/launches_small.csv | python -c "
import csv,sys
for x in csv.DictReader(sys.stdin):
  if x.get('Metric Name')=='gpu__time_duration.sum': print(x['Kernel Name'][:60], x['Grid Size'], x['Block Size'], x['Metric Value'])
"
