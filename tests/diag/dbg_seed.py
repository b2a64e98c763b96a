"""Debug: compare one random instance (test_random_small_instances recipe) on both plans."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))), "tests"))
import numpy as np
import oracle, workloads
from helpers import to_oracle
import paper_2511_15629_b200 as E

seed = int(sys.argv[1]) if len(sys.argv) > 1 else 34
kind = [workloads.PAYOFF_LINEAR, workloads.PAYOFF_LINEAR_MINUS_G, workloads.PAYOFF_TABLE][seed % 3]
inst = workloads.random_instance(seed, S_max=40 if seed % 2 else 600, T=4 + seed % 3, K=1 + seed % 4)
S, A = oracle.dims(to_oracle(inst))
inst.payoff_kind = kind
if kind == workloads.PAYOFF_LINEAR_MINUS_G:
    inst.g = workloads.random_g(seed, A, 20.0)
elif kind == workloads.PAYOFF_TABLE:
    inst.g = workloads.random_table(seed, inst.T, inst.K, A)
pr = to_oracle(inst)
ref = oracle.backward(pr)
print("T K S A", inst.T, inst.K, S, A, "rank1", inst.P is None, "kind", kind)
print("g", inst.g if kind == 1 else None)
for persist in (False, True):
    for brute in (False, True):
        with E.Solver(inst, persist=persist, force_brute=brute) as s:
            J = s.backward()
            print(f"persist={persist} brute={brute} kind={s.stencil_kind} J ok={J == ref.J}")
            for t in range(inst.T, 0, -1):
                V, W = s.values(t)
                pol = s.policy(t)
                dv = np.argwhere(V != ref.V[t - 1]); dw = np.argwhere(W != ref.W[t - 1]); dp = np.argwhere(pol != ref.pol[t - 1])
                if len(dv) or len(dw) or len(dp):
                    print(f"  t={t}: W diffs {len(dw)} V diffs {len(dv)} {dv[:4].tolist()} pol diffs {len(dp)} {dp[:4].tolist()}")
                    if len(dv):
                        k, i = dv[0]
                        print("   V", V[k, i], ref.V[t-1][k, i], "pol", pol[k, i], ref.pol[t-1][k, i])
                    break
