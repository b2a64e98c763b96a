"""Warm per-launch kernel times and chain time per stage for a cfg4-shaped problem (T=64)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2511_15629_b200 as E
import workloads

inst = workloads.cfg4(T=64)
s = E.Solver(inst, keep_values=True)
for _ in range(3):
    s.backward()
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(5):
    s.backward()
torch.cuda.synchronize()
ms = (time.perf_counter() - t0) / 5 * 1e3
print(f"cfg4-shaped T=64: backward {ms:.3f} ms ({ms / 64 * 1e3:.2f} us/stage) | warm us/launch: contract "
      f"{E.esdp_debug_time(s.ctx, 0):.2f} stencil {E.esdp_debug_time(s.ctx, 1):.2f} brute {E.esdp_debug_time(s.ctx, 2):.2f}")
