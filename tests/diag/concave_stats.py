"""Exact concavity of the oracle's W over the window stencil's tile columns (diagnostic, CPU): math.fsum sign of W[j-1] + W[j+1] - 2 W[j]."""
import sys, math, numpy as np
import os; R = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))); sys.path.insert(0, R); sys.path.insert(0, os.path.join(R, 'tests'))
import oracle, workloads
from helpers import to_oracle
for name, inst in [("cfg2", workloads.cfg2(T=24)), ("t3", workloads.table3(hours=100.0, delta=0.01, T=6))]:
    pr = to_oracle(inst)
    ref = oracle.backward(pr, nthreads=16)
    S = ref.W.shape[2]
    tot = exact = 0; worst = []
    for t in range(1, inst.T):
        rows = ref.W[t - 1] if inst.P is not None else ref.W[t - 1][:1]
        for W in rows:
            # second differences exactly: sign of a + b - 2c via fsum
            d = np.array([math.fsum([W[j-1], W[j+1], -2.0 * W[j]]) for j in range(1, S - 1)])
            for i0 in range(0, S, 256):
                lo = max(0, i0 - 105); hi = min(S - 1, i0 + 255 + 105)
                seg = d[max(lo, 1) - 1: hi - 1]
                tot += 1
                m = seg.max() if len(seg) else 0.0
                exact += m <= 0
                worst.append(m / max(1.0, np.abs(W).max()))
    w = np.array(worst)
    print(name, "tiles", tot, "exactly concave", exact / tot, "max rel defect quantiles", np.quantile(w, [0.5, 0.9, 0.99, 1.0]))
