"""Simulation kernel time after a backward pass, with and without keeping V/W (L2 pollution check)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2511_15629_b200 as E
import workloads

inst = workloads.cfg2()
for keep in (True, False):
    s = E.Solver(inst, keep_values=keep)
    out = torch.empty(65536, dtype=torch.float64, device="cuda")
    st = torch.cuda.Stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for rep in range(6):
        E.esdp_backward_async(s.ctx, st.cuda_stream)
        e0.record(st)
        E.esdp_simulate_dev(s.ctx, 65536, rep, out.data_ptr(), st.cuda_stream)
        e1.record(st)
        st.synchronize()
        ts.append(e0.elapsed_time(e1))
    # second sim right after the first (pol hot in L2)
    e0.record(st); E.esdp_simulate_dev(s.ctx, 65536, 99, out.data_ptr(), st.cuda_stream); e1.record(st); st.synchronize()
    print(f"keep={keep}: sim after backward {min(ts[2:]):.3f} ms; sim again (hot) {e0.elapsed_time(e1):.3f} ms")
    s.close()
