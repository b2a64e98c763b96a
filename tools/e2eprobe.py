"""Device time vs wall time of the pipelined e2e loop (diagnostic)."""
import ctypes, os, sys, time
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
nv = torch.empty(n, dtype=torch.int32, device="cuda"); vert = torch.empty(n * A, dtype=torch.int16, device="cuda")
pr = torch.empty(n * A, dtype=torch.float64, device="cuda")
mode = sys.argv[1] if len(sys.argv) > 1 else "load"
if "nobids" not in mode:
    E.esdp_set_bid_requests(s.ctx, req, A, nv.data_ptr(), vert.data_ptr(), None, pr.data_ptr())
stream = torch.cuda.Stream(); sp = stream.cuda_stream
lam_h = torch.from_numpy(np.ascontiguousarray(inst.lam)).pin_memory()
P_h = torch.from_numpy(np.ascontiguousarray(inst.P)).pin_memory()
pi_h = torch.from_numpy(np.ascontiguousarray(inst.pi)).pin_memory()
dp = ctypes.POINTER(ctypes.c_double); as_p = lambda t: ctypes.cast(t.data_ptr(), dp)
side = torch.cuda.Stream()
P_dev = torch.empty_like(P_h, device="cuda")
st_d = torch.zeros(2, dtype=torch.float64, device="cuda")
st_side = torch.zeros(1024, dtype=torch.float64, device="cuda")
side_ev, main_ev = torch.cuda.Event(), torch.cuda.Event()
side_hi = torch.cuda.Stream(priority=-5)
evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(13)]
mid = [torch.cuda.Event(enable_timing=True) for _ in range(13)]
for j in range(13):
    evs[j][0].record(stream)
    E.lib.esdp_backward_async(s.ctx, sp)
    mid[j].record(stream)
    main_ev.record(stream)
    if mode == "load":
        assert E.lib.esdp_load_async(s.ctx, as_p(lam_h), as_p(P_h), as_p(pi_h), None) == 0
    if mode == "dma":
        with torch.cuda.stream(side):
            P_dev.copy_(P_h, non_blocking=True)
    if mode.endswith("kernel") and mode != "dmakernel":   # one small kernel on another stream while the backward runs
        with torch.cuda.stream(side):
            st_side.add_(1.0)
    if mode == "evrec":     # an event record on another stream
        side_ev.record(side)
    if mode == "evwait":    # another stream waits for the main stream (cross-stream dependency), then a DMA
        side.wait_event(main_ev)
        with torch.cuda.stream(side):
            P_dev.copy_(P_h, non_blocking=True)
    if mode == "kernelhi":  # the small kernel on a high-priority stream
        with torch.cuda.stream(side_hi):
            st_side.add_(1.0)
    if mode == "dmakernel":
        with torch.cuda.stream(side):
            P_dev.copy_(P_h, non_blocking=True)
            st_side.add_(1.0)
    E.lib.esdp_simulate_async(s.ctx, 65536, 99 + j, ctypes.c_void_p(st_d.data_ptr()), sp)
    evs[j][1].record(stream)
torch.cuda.synchronize()
t0 = time.perf_counter()
for j in range(10):
    evs[j][0].record(stream)
    E.lib.esdp_backward_async(s.ctx, sp)
    mid[j].record(stream)
    main_ev.record(stream)
    if mode == "load":
        assert E.lib.esdp_load_async(s.ctx, as_p(lam_h), as_p(P_h), as_p(pi_h), None) == 0
    if mode == "dma":
        with torch.cuda.stream(side):
            P_dev.copy_(P_h, non_blocking=True)
    if mode.endswith("kernel") and mode != "dmakernel":   # one small kernel on another stream while the backward runs
        with torch.cuda.stream(side):
            st_side.add_(1.0)
    if mode == "evrec":     # an event record on another stream
        side_ev.record(side)
    if mode == "evwait":    # another stream waits for the main stream (cross-stream dependency), then a DMA
        side.wait_event(main_ev)
        with torch.cuda.stream(side):
            P_dev.copy_(P_h, non_blocking=True)
    if mode == "kernelhi":  # the small kernel on a high-priority stream
        with torch.cuda.stream(side_hi):
            st_side.add_(1.0)
    if mode == "dmakernel":
        with torch.cuda.stream(side):
            P_dev.copy_(P_h, non_blocking=True)
            st_side.add_(1.0)
    E.lib.esdp_simulate_async(s.ctx, 65536, 99 + j, ctypes.c_void_p(st_d.data_ptr()), sp)
    evs[j][1].record(stream)
torch.cuda.synchronize()
wall = (time.perf_counter() - t0) / 10 * 1e3
dev = np.mean([evs[j][0].elapsed_time(evs[j][1]) for j in range(10)])
gap = np.mean([evs[j][1].elapsed_time(evs[j + 1][0]) for j in range(9)])
bw = np.mean([evs[j][0].elapsed_time(mid[j]) for j in range(10)])
print(f"mode={mode}: wall {wall:.3f} ms/step, device {dev:.3f} ms/step (backward {bw:.3f}, sim {dev - bw:.3f}), gap {gap:.3f} ms")
