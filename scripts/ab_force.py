"""A/B: k_force_fast with partials out (+ the update's reduce) vs the fused in-kernel reduction, N = 2^20."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2411_18889_b200 as b2  # noqa: E402
from paper_2411_18889_b200 import _lib  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
lib = b2.load()
pos, _ = b2.plummer(n, 42)
acc = torch.empty_like(pos)
nch = lib.b2_calc_acc_nchunks(n, 0)
part = torch.empty((nch * n, 4), device="cuda")
ws = b2.workspace(n, n)
sh = _lib.stream_handle()
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")


def unfused():
    lib.b2_calc_acc_partials(n, pos.data_ptr(), n, pos.data_ptr(), 2 ** -6, 0, part.data_ptr(), sh)


def fused():
    lib.b2_calc_acc(n, pos.data_ptr(), acc.data_ptr(), n, pos.data_ptr(), 2 ** -6, 0, ws.data_ptr(), ws.numel(), sh)


for f in (unfused, fused):
    f()
res = {"unfused": [], "fused": []}
for rep in range(4):
    for name, f in (("unfused", unfused), ("fused", fused)):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        f()
        e1.record()
        torch.cuda.synchronize()
        res[name].append(e0.elapsed_time(e1))
for k, v in res.items():
    print(k, " ".join(f"{x:.2f}" for x in v), "min %.2f" % min(v))
