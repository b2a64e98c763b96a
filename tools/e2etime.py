"""Host-side phase times of the end-to-end step (diagnostic): load_async / backward / simulate."""
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
dp = ctypes.POINTER(ctypes.c_double)
as_p = lambda t: ctypes.cast(t.data_ptr(), dp)
J = ctypes.c_double(); m = ctypes.c_double(); v = ctypes.c_double()
acc = np.zeros(4)
for j in range(13):
    t0 = time.perf_counter()
    assert E.lib.esdp_load_async(s.ctx, as_p(lam_h), as_p(P_h), as_p(pi_h), None) == 0
    t1 = time.perf_counter()
    assert E.lib.esdp_backward(s.ctx, None, ctypes.byref(J)) == 0
    t2 = time.perf_counter()
    assert E.lib.esdp_simulate(s.ctx, 65536, 99 + j, ctypes.byref(m), ctypes.byref(v), None) == 0
    t3 = time.perf_counter()
    if j >= 3:
        acc += np.array([t1 - t0, t2 - t1, t3 - t2, t3 - t0]) * 1e3
print("ms per step: load_async %.3f  backward %.3f  simulate %.3f  total %.3f" % tuple(acc / 10))
for j in range(3):
    t0 = time.perf_counter()
    assert E.lib.esdp_load(s.ctx, as_p(lam_h), as_p(P_h), as_p(pi_h), None) == 0
    t1 = time.perf_counter()
print("sync esdp_load %.3f ms" % ((t1 - t0) * 1e3))
