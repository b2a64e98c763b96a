"""Host time of esdp_load_async (validation, slice dedupe, chunked H2D enqueue) on cfg2 (diagnostic)."""
import ctypes, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2511_15629_b200 as E
import workloads

inst = workloads.cfg2()
s = E.Solver(inst, keep_values=True)
lam_h = torch.from_numpy(np.ascontiguousarray(inst.lam)).pin_memory()
P_h = torch.from_numpy(np.ascontiguousarray(inst.P)).pin_memory()
pi_h = torch.from_numpy(np.ascontiguousarray(inst.pi)).pin_memory()
dp = ctypes.POINTER(ctypes.c_double); as_p = lambda t: ctypes.cast(t.data_ptr(), dp)
ts = []
for j in range(12):
    E.lib.esdp_backward_async(s.ctx, None)
    t0 = time.perf_counter()
    assert E.lib.esdp_load_async(s.ctx, as_p(lam_h), as_p(P_h), as_p(pi_h), None) == 0
    ts.append(time.perf_counter() - t0)
    torch.cuda.synchronize()
print("esdp_load_async host time (ms): median %.3f min %.3f" % (1e3 * np.median(ts[2:]), 1e3 * min(ts[2:])))
