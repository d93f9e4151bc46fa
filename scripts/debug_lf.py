import ctypes, os, sys
import torch
import paper_2411_18889_b200 as b2
from paper_2411_18889_b200 import _lib
lib = b2.load()
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
pos, vel = b2.plummer(n, 42)
acc = torch.empty_like(pos)
ws = torch.empty(int(lib.b2_leapfrog_workspace_bytes(n, 0)), dtype=torch.uint8, device="cuda")
sh = _lib.stream_handle()
print("partials", lib.b2_calc_acc_partials(n, pos.data_ptr(), n, pos.data_ptr(), 0.01, 0, ws.data_ptr(), sh))
print("leapfrog init", lib.b2_leapfrog(n, pos.data_ptr(), vel.data_ptr(), acc.data_ptr(), 0.01, 0.01, 0, 4, ws.data_ptr(), ws.numel(), sh))
print("leapfrog 2", lib.b2_leapfrog(n, pos.data_ptr(), vel.data_ptr(), acc.data_ptr(), 0.01, 0.01, 2, 0, ws.data_ptr(), ws.numel(), sh))
torch.cuda.synchronize()
which = ctypes.c_int(0)
print("fault", lib.b2_fault_status(sh, 0, ctypes.byref(which)), which.value)
