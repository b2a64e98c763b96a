"""Task trace of the persistent dataflow kernel (diagnostic; needs `make -B EXTRA=-DESDP_DF_TRACE`):
python tools/dftrace.py [cfg2|cfg2-rank1] -> per-kind task run times, busy CTAs, stage cadence."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2511_15629_b200 as E
import workloads

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
inst = workloads.cfg2(rank1=cfg.endswith("rank1"))
s = E.Solver(inst, keep_values=True, persist=True)
for _ in range(3):
    s.backward()
torch.cuda.synchronize()
n = 1 << 18
buf = np.zeros((n, 4), np.uint64)
E.lib.esdp_df_trace.argtypes = [ctypes.c_void_p, ctypes.c_int]
assert E.lib.esdp_df_trace(buf.ctypes.data, n) == 0
np.save("gpurun_out/dftrace_%s.npy" % cfg, buf)
ok = (buf[:, 0] > 0) & (buf[:, 2] > 0)
idx = np.nonzero(ok)[0]
tr = buf[ok].astype(np.float64)
t0 = tr[:, 0].min()
pop, start, done = (tr[:, 0] - t0) / 1e3, (tr[:, 1] - t0) / 1e3, (tr[:, 2] - t0) / 1e3
print("tasks", ok.sum(), "span %.1f us, %.2f us/stage" % (done.max(), done.max() / inst.T))
run = done - pop
ev = np.concatenate([pop, done]); sg = np.concatenate([np.ones(len(pop)), -np.ones(len(pop))])
o = np.argsort(ev); c = np.cumsum(sg[o]); tt = ev[o]
print("busy CTAs: max %d, time-weighted mean %.1f; SMs used %d" % (c.max(), np.sum(c[:-1] * np.diff(tt)) / (tt[-1] - tt[0]),
                                                                    len(np.unique(tr[:, 3]))))
K = inst.K
S = 1001
ntc = (S + 255) // 256
nS = K * ntc
period = None
# infer the period from the number of tasks per stage: nS + nE
for p in range(nS, nS + 2000):
    if (ok.sum() - 1 - nS) % p == 0 and (ok.sum() - 1 + (p - nS)) // p == inst.T:
        period = p
        break
print("period", period)
pos = idx % period
st = idx // period
isS = pos < 0
# S entries: the pattern starts each tile with K S tasks
print("run us: all mean %.2f p50 %.2f p90 %.2f" % (run.mean(), np.median(run), np.percentile(run, 90)))
ends = np.array([done[st == k].max() for k in range(inst.T)])
print("per-period end deltas (us): first 5", np.round(np.diff(ends[:6]), 2), "median", np.median(np.diff(ends)))
