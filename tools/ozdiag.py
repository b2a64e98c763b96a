import sys, os
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import numpy as np, torch
import paper_2511_15629_b200 as E, workloads, oracle
from helpers import to_oracle
for T in (2, 3, 10):
    insts = workloads.cfg5_instances([0, 300, 777, 1023], T=T, K=100)
    with E.Batch(insts, ozaki=True) as b:
        J = b.backward()
        for m, inst in enumerate(insts):
            pr = to_oracle(inst); ref = oracle.backward(pr, nthreads=16)
            V1 = b.value1(m); d = np.abs(V1 - ref.V[0])
            k, i = np.unravel_index(np.argmax(d / np.maximum(1, np.abs(ref.V[0]))), d.shape)
            print(T, m, "J rel %.2e" % (abs(J[m]-ref.J)/abs(ref.J)), "V1 max abs %.2e" % d.max(), "at", k, i, "ref %.6g" % ref.V[0][k, i],
                  "V1 max %.3g" % ref.V[0].max(), "Wmax %.3g" % ref.W[0].max())
            # product check on the oracle's own V_2 -> W_1
            if T >= 2:
                S = ref.V.shape[2]
                P1 = np.ascontiguousarray(inst.P[0]); V2 = np.ascontiguousarray(ref.V[1])
                Pd = torch.from_numpy(P1).cuda(); Vd = torch.from_numpy(V2).cuda(); Wd = torch.zeros_like(Vd)
                E.expectation_dev(Pd.data_ptr(), Vd.data_ptr(), Wd.data_ptr(), 100, 100, S, S, S, 1)
                torch.cuda.synchronize(); W1 = Wd.cpu().numpy()
                ex = P1.astype(np.longdouble) @ V2.astype(np.longdouble)
                print("   product W_1 from oracle V_2: max rel err %.2e, oracle fma-chain rel err %.2e" % (
                    float(np.max(np.abs(W1 - ex) / np.maximum(1, np.abs(ex)))), float(np.max(np.abs(ref.W[0] - ex) / np.maximum(1, np.abs(ex))))))
