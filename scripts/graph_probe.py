# Probe: CUDA-graph replay of Leapfrog.step(32) vs direct calls at mid N (DESIGN.md size table).
import sys; sys.path.insert(0, '.')
import torch, paper_2411_18889_b200 as b2
for n in (8192, 16384, 32768):
    for graphs in (False, True):
        pos, vel = b2.plummer(n, 42)
        lf = b2.Leapfrog(pos, vel, 2.0**-6, 2.0**-7, graphs=graphs)
        lf.step(8); torch.cuda.synchronize()
        e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        e[0].record(); lf.step(8); lf.step(8); lf.step(8); lf.step(8); e[1].record(); torch.cuda.synchronize()
        print(f'n={n} Leapfrog(graphs={graphs}).step(8): {e[0].elapsed_time(e[1]) / 32 * 1e3:.1f} us/step')
    pos, vel = b2.plummer(n, 42)
    lf = b2.Leapfrog(pos, vel, 2.0**-6, 2.0**-7)
    lf.step(4); torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record(); lf.step(32); ev[1].record(); torch.cuda.synchronize()
    direct = ev[0].elapsed_time(ev[1]) / 32
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        lf.step(2)
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        lf.step(32)
    g.replay(); torch.cuda.synchronize()
    ev[0].record(); g.replay(); ev[1].record(); torch.cuda.synchronize()
    graph = ev[0].elapsed_time(ev[1]) / 32
    print(f"n={n} direct {direct*1e3:.1f} us/step graph {graph*1e3:.1f} us/step ({n*n/graph/1e6:.0f} Ginter/s)")
