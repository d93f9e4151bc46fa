import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, paper_2411_18889_b200 as b2
for n in (8192, 16384, 1 << 15):
    pos, _ = b2.plummer_numpy(n, 8)
    p = torch.from_numpy(pos).cuda()
    full = b2.accelerations(p, 2 ** -6)
    for parts in (2, 4):
        sl = n // parts
        bad = 0
        for r in range(parts):
            part = b2.accelerations(p[r * sl:(r + 1) * sl].contiguous(), 2 ** -6, p)
            bad += int((part != full[r * sl:(r + 1) * sl]).any(1).sum())
        print(n, parts, "mismatching rows", bad)
