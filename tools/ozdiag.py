"""Accuracy of the Ozaki tcgen05 expectation plan (ESDP_CONTRACT_OZAKI) end to end against the FP64 oracle:
python tools/ozdiag.py [T] -> per instance: J relative error, worst V_1 error relative to max(1, |V|) and to the
row maximum, policy differences (diagnostic; DESIGN.md §5 NEXT-4)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import paper_2511_15629_b200 as E
import workloads
import oracle
from helpers import to_oracle

T = int(sys.argv[1]) if len(sys.argv) > 1 else 288
insts = workloads.cfg5_instances([0, 300, 777, 1023], T=T, K=100)
with E.Batch(insts, ozaki=True) as b:
    assert b.plan == 2
    J = b.backward()
    for m, inst in enumerate(insts):
        ref = oracle.backward(to_oracle(inst), nthreads=os.cpu_count() or 1)
        V1 = b.value1(m)
        d = np.abs(V1 - ref.V[0])
        rel1 = float(np.max(d / np.maximum(1.0, np.abs(ref.V[0]))))
        relrow = float(np.max(d / np.maximum(1e-300, np.abs(ref.V[0]).max(axis=1, keepdims=True))))
        npol = sum(int(np.sum(b.policy(m, t) != ref.pol[t - 1])) for t in range(1, T + 1))
        print(f"T={T} instance {m}: J rel {abs(J[m] - ref.J) / abs(ref.J):.2e}, V_1 max |d|/max(1,|V|) {rel1:.2e}, "
              f"/ row max {relrow:.2e}, policy entries differing {npol} of {T * inst.K * b.S}", flush=True)
