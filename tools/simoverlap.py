"""Timing experiment (diagnostic; the numbers it prints are not results): the cfg2 step with the simulation of
step j on a second stream, overlapping the backward of step j+1, against the serial step.  The library has
ONE policy buffer, so the overlapped simulation reads a policy that the next backward is rewriting: its
output is meaningless here; only the device time per step is of interest (would a policy double buffer pay?).
    python tools/simoverlap.py"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2511_15629_b200 as E
import workloads

inst = workloads.cfg2()
s = E.Solver(inst, keep_values=True)
T, S, A, K = s.T, s.S, s.A, s.K
tt, ii = np.meshgrid(np.arange(1, T + 1, dtype=np.int32), np.arange(S, dtype=np.int32), indexing="ij")
req = np.stack([tt.ravel(), ii.ravel(), np.full(T * S, K // 2, np.int32)], 1).astype(np.int32)
n = req.shape[0]
dev = torch.device("cuda")
nv = torch.empty(n, dtype=torch.int32, device=dev); vert = torch.empty(n * A, dtype=torch.int16, device=dev)
pr = torch.empty(n * A, dtype=torch.float64, device=dev)
E.esdp_set_bid_requests(s.ctx, req, A, nv.data_ptr(), vert.data_ptr(), None, pr.data_ptr())
main, side = torch.cuda.Stream(), torch.cuda.Stream()
st = torch.zeros(2, dtype=torch.float64, device=dev)
ev_done = [torch.cuda.Event() for _ in range(64)]
t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def run(overlap, steps=20, warm=4):
    for j in range(warm + steps):
        if j == warm:
            torch.cuda.synchronize()
            t0.record(main)
        assert E.lib.esdp_backward_async(s.ctx, main.cuda_stream) == 0
        if overlap:
            ev_done[j].record(main)
            side.wait_event(ev_done[j])
            assert E.lib.esdp_simulate_async(s.ctx, 65536, 7 + j, ctypes.c_void_p(st.data_ptr()), side.cuda_stream) == 0
        else:
            assert E.lib.esdp_simulate_async(s.ctx, 65536, 7 + j, ctypes.c_void_p(st.data_ptr()), main.cuda_stream) == 0
    main.wait_stream(side)
    t1.record(main)
    torch.cuda.synchronize()
    return t0.elapsed_time(t1) / steps


for overlap in (False, True, False, True):
    print(f"{'overlapped' if overlap else 'serial'}: {run(overlap):.3f} ms per step")
