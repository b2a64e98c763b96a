"""Sampling-table guide density (ESDP_GUIDE_RATIO buckets per state) against the table build and the
simulation (diagnostic).  Run once per ratio (the density is fixed at context creation):
    ESDP_GUIDE_RATIO=4 python tools/guidesweep.py
Prints, for cfg2 and 65,536 paths: the simulation after a fresh upload (lazy table build + simulation)
and the simulation alone (tables current), both as warm per-call device times."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2511_15629_b200 as E
import workloads

inst = workloads.cfg2()
s = E.Solver(inst, keep_values=False)
stream = torch.cuda.Stream(); sp = stream.cuda_stream
lam_h = torch.from_numpy(np.ascontiguousarray(inst.lam)).pin_memory()
P_h = torch.from_numpy(np.ascontiguousarray(inst.P)).pin_memory()
pi_h = torch.from_numpy(np.ascontiguousarray(inst.pi)).pin_memory()
dp = ctypes.POINTER(ctypes.c_double); as_p = lambda t: ctypes.cast(t.data_ptr(), dp)
st_d = torch.zeros(2, dtype=torch.float64, device="cuda")
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
stats = {}
for fresh in (True, False):
    ts = []
    for j in range(8):
        if fresh:
            assert E.lib.esdp_load_async(s.ctx, as_p(lam_h), as_p(P_h), as_p(pi_h), None) == 0
        assert E.lib.esdp_backward_async(s.ctx, sp) == 0
        stream.synchronize()
        ev[0].record(stream)
        assert E.lib.esdp_simulate_async(s.ctx, 65536, 99 + j, ctypes.c_void_p(st_d.data_ptr()), sp) == 0
        ev[1].record(stream)
        stream.synchronize()
        if j >= 3:
            ts.append(ev[0].elapsed_time(ev[1]))
    stats["after upload" if fresh else "tables current"] = np.median(ts)
    m = float(st_d[0])
print(f"ratio {os.environ.get('ESDP_GUIDE_RATIO', 'default')}: " +
      ", ".join(f"{k} {v * 1e3:.1f} us" for k, v in stats.items()) + f"; mean profit {m:.6f}")
