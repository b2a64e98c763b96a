"""Small end-to-end run for compute-sanitizer: every kernel kind on cfg1 (window + brute stencils, DMMA + DFMA
expectation, bid curves on demand and fused into the graph, simulation), a rank-1 instance, a batch on the
Ozaki tcgen05 plan."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2511_15629_b200 as E
import workloads

for inst in (workloads.cfg1("b"), workloads.cfg1("a", rank1=True), workloads.cfg2(T=3, K=9)):
    for kw in (dict(), dict(force_brute=True), dict(dmma=False)):
        with E.Solver(inst, **kw) as s:
            J = s.backward()
            req = np.array([(t, i, k) for t in (1, inst.T) for i in range(0, s.S, 13) for k in range(inst.K)])
            s.bidcurves(req)
            n = len(req); cap = s.A
            nv = torch.zeros(n, dtype=torch.int32, device="cuda")
            vt = torch.zeros(cap * n, dtype=torch.int16, device="cuda")
            pr = torch.zeros(cap * n, dtype=torch.float64, device="cuda")
            E.esdp_set_bid_requests(s.ctx, req, cap, nv.data_ptr(), vt.data_ptr(), None, pr.data_ptr())
            s.backward()
            s.simulate(256, 1)
            print(inst.name, kw, "J=%.6f" % J, flush=True)
with E.Batch(workloads.cfg5_instances([0, 511, 1023], T=4, K=16), ozaki=True) as b:
    b.backward()
    print("batch ozaki plan", b.plan, flush=True)
print("sanitize run ok")
