"""The bench's e2e loop (bench.py run_ours) on cfg2 with host-side timestamps per call (diagnostic)."""
import ctypes, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2511_15629_b200 as E
import workloads

inst = workloads.cfg2()
dev = torch.device("cuda")
solver = E.Solver(inst, keep_values=True)
T, S, A, K = solver.T, solver.S, solver.A, solver.K
tt, ii = np.meshgrid(np.arange(1, T + 1, dtype=np.int32), np.arange(S, dtype=np.int32), indexing="ij")
req = np.stack([tt.ravel(), ii.ravel(), np.full(T * S, K // 2, np.int32)], 1).astype(np.int32)
n = req.shape[0]
nv = torch.empty(n, dtype=torch.int32, device=dev); vert = torch.empty(n * A, dtype=torch.int16, device=dev)
pr = torch.empty(n * A, dtype=torch.float64, device=dev)
if "nobids" not in sys.argv:
    E.esdp_set_bid_requests(solver.ctx, req, A, nv.data_ptr(), vert.data_ptr(), None, pr.data_ptr())
stream = torch.cuda.Stream(); sp = stream.cuda_stream
lam_h = torch.from_numpy(np.ascontiguousarray(inst.lam)).pin_memory()
P_h = torch.from_numpy(np.ascontiguousarray(inst.P)).pin_memory()
pi_h = torch.from_numpy(np.ascontiguousarray(inst.pi)).pin_memory()
dp = ctypes.POINTER(ctypes.c_double); as_p = lambda t: ctypes.cast(t.data_ptr(), dp)
load = lambda: E.lib.esdp_load_async(solver.ctx, as_p(lam_h), as_p(P_h), as_p(pi_h), None)
J_h = torch.zeros(2, dtype=torch.float64).pin_memory()
st_h = torch.zeros((2, 2), dtype=torch.float64).pin_memory()
st_d = torch.zeros((2, 2), dtype=torch.float64, device=dev)
done = [torch.cuda.Event(), torch.cuda.Event()]
dev_ev = [torch.cuda.Event(enable_timing=True) for _ in range(40)]
assert load() == 0
hx = {"backward": 0.0, "load": 0.0, "objective": 0.0, "simulate": 0.0, "read": 0.0}
def read(j):
    t = time.perf_counter(); done[j % 2].synchronize(); hx["read"] += time.perf_counter() - t
nstep, warm = 13, 3
for j in range(nstep):
    if j == warm:
        read(j - 1); torch.cuda.synchronize(); t0 = time.perf_counter(); hx = dict.fromkeys(hx, 0.0)
    dev_ev[j].record(stream)
    t = time.perf_counter(); assert E.lib.esdp_backward_async(solver.ctx, sp) == 0; hx["backward"] += time.perf_counter() - t
    if j + 1 < nstep:
        t = time.perf_counter(); assert load() == 0; hx["load"] += time.perf_counter() - t
    t = time.perf_counter(); assert E.lib.esdp_objective_async(solver.ctx, ctypes.c_void_p(J_h[j % 2:].data_ptr()), sp) == 0; hx["objective"] += time.perf_counter() - t
    t = time.perf_counter(); assert E.lib.esdp_simulate_async(solver.ctx, 65536, 99 + j, ctypes.c_void_p(st_d[j % 2].data_ptr()), sp) == 0
    with torch.cuda.stream(stream):
        st_h[j % 2].copy_(st_d[j % 2], non_blocking=True)
    hx["simulate"] += time.perf_counter() - t
    done[j % 2].record(stream)
    if j > 0 and j != warm:
        read(j - 1)
read(nstep - 1)
wall = (time.perf_counter() - t0) / (nstep - warm) * 1e3
devs = [dev_ev[j].elapsed_time(dev_ev[j + 1]) for j in range(warm, nstep - 1)]
print(f"e2e wall {wall:.3f} ms/step; device step-to-step {np.mean(devs):.3f} ms; host per step (ms): " +
      ", ".join(f"{k} {v / (nstep - warm) * 1e3:.3f}" for k, v in hx.items()))
