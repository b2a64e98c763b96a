"""Warm per-kernel launch times on cfg2 (diagnostic): python tools/ktime.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2511_15629_b200 as E
import workloads
import time

inst = workloads.cfg2()
for keep in (True,):
    s = E.Solver(inst, keep_values=keep)
    s.backward()
    names = ["contract", "stencil(" + ("window" if s.stencil_kind else "brute") + ")", "stencil(brute)", "objective"]
    for w in range(4):
        print(f"{names[w]:18s} {E.esdp_debug_time(s.ctx, w, 200):8.2f} us/launch")
    for _ in range(3):
        s.backward()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(10):
        s.backward()
    torch.cuda.synchronize()
    print(f"backward graph: {(time.perf_counter() - t0) / 10 * 1e3:.3f} ms  ({(time.perf_counter() - t0) / 10 / inst.T * 1e6:.2f} us/stage)")
    s.close()
