"""The backward right after an input-slot switch (a load) against a repeat on the same slot (diagnostic):
per step load -> backward (new slot) -> backward (same slot) -> simulate, device-timed each."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2511_15629_b200 as E
import workloads

inst = workloads.cfg2()
s = E.Solver(inst, keep_values="nokeep" not in sys.argv)
stream = torch.cuda.Stream(); sp = stream.cuda_stream
lam_h = torch.from_numpy(np.ascontiguousarray(inst.lam)).pin_memory()
P_h = torch.from_numpy(np.ascontiguousarray(inst.P)).pin_memory()
pi_h = torch.from_numpy(np.ascontiguousarray(inst.pi)).pin_memory()
dp = ctypes.POINTER(ctypes.c_double); as_p = lambda t: ctypes.cast(t.data_ptr(), dp)
ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(10)]
res = []
for j in range(10):
    assert E.lib.esdp_load_async(s.ctx, as_p(lam_h), as_p(P_h), as_p(pi_h), None) == 0
    torch.cuda.synchronize()   # the upload has landed: only the switch differs
    ev[j][0].record(stream)
    assert E.lib.esdp_backward_async(s.ctx, sp) == 0
    ev[j][1].record(stream)
    assert E.lib.esdp_backward_async(s.ctx, sp) == 0
    ev[j][2].record(stream)
    torch.cuda.synchronize()
    if j >= 3:
        res.append((ev[j][0].elapsed_time(ev[j][1]), ev[j][1].elapsed_time(ev[j][2])))
r = np.median(np.array(res), axis=0)
print(f"{' '.join(sys.argv[1:]) or 'keep'}: backward after a slot switch {r[0]:.3f} ms, repeated on the same slot {r[1]:.3f} ms")
