"""Bid-curve kernel alone (diagnostic): every (t, i) curve at k = K/2 of a short horizon of cfg2 or cfg4,
one esdp_bidcurves_dev launch over all of them, warm device time per launch and the average hull size.
    python tools/bidprobe.py cfg2|cfg4 [T]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2511_15629_b200 as E
import workloads

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
T = int(sys.argv[2]) if len(sys.argv) > 2 else 36
inst = workloads.cfg2(T=T) if name == "cfg2" else workloads.cfg4(T=T)
s = E.Solver(inst, keep_values=True)
s.backward()
S, A, K = s.S, s.A, s.K
tt, ii = np.meshgrid(np.arange(1, T + 1, dtype=np.int32), np.arange(S, dtype=np.int32), indexing="ij")
req = np.stack([tt.ravel(), ii.ravel(), np.full(T * S, K // 2, np.int32)], 1).astype(np.int32)
n = req.shape[0]
dev = torch.device("cuda")
req_d = torch.from_numpy(req).to(dev)
nv = torch.empty(n, dtype=torch.int32, device=dev)
vert = torch.empty(n * A, dtype=torch.int16, device=dev)
price = torch.empty(n * A, dtype=torch.float64, device=dev)
stream = torch.cuda.Stream()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ts = []
for j in range(8):
    ev[0].record(stream)
    E.esdp_bidcurves_dev(s.ctx, n, req_d.data_ptr(), A, nv.data_ptr(), vert.data_ptr(), None, price.data_ptr(), stream)
    ev[1].record(stream)
    stream.synchronize()
    if j >= 3:
        ts.append(ev[0].elapsed_time(ev[1]))
us = float(np.median(ts)) * 1e3
print(f"{name} T={T}: {n} curves, A={A}, mean hull {float(nv.float().mean()):.1f} vertices: {us:.1f} us per launch "
      f"({n / us:.1f} curves/us)")
