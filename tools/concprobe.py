"""Cost of one small operation on another stream while the backward graph runs (diagnostic): the cfg2
backward (KEEP_VALUES, no bid curves, synchronized between steps) device-timed alone and with a one-block
kernel, a 1 KB / 4 MB pinned H2D copy or an event record on a second stream, right after the graph's launch
or 1 ms into it.  (In this synchronized setting none of them cost anything measurable; in the pipelined loop of
tools/e2eprobe.py a foreign kernel costs the graph ~0.22 ms -- DESIGN.md §7.)"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2511_15629_b200 as E
import workloads

inst = workloads.cfg2()
s = E.Solver(inst, keep_values=True)
stream = torch.cuda.Stream(); sp = stream.cuda_stream
lo, hi = torch.cuda.Stream(priority=0), torch.cuda.Stream(priority=-5)
x = torch.zeros(1024, dtype=torch.float64, device="cuda")
small_h = torch.zeros(128, dtype=torch.float64).pin_memory()       # 1 KB
big_h = torch.zeros(1 << 19, dtype=torch.float64).pin_memory()     # 4 MB
small_d = torch.zeros(128, dtype=torch.float64, device="cuda")
big_d = torch.zeros(1 << 19, dtype=torch.float64, device="cuda")
side_ev = torch.cuda.Event()
WHAT = "kernel"

def side_work(side):
    with torch.cuda.stream(side):
        if WHAT == "kernel":
            x.add_(1.0)
        elif WHAT == "h2d_1KB":
            small_d.copy_(small_h, non_blocking=True)
        elif WHAT == "h2d_4MB":
            big_d.copy_(big_h, non_blocking=True)
        elif WHAT == "event":
            side_ev.record(side)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]

def run(where, side):
    ts = []
    for j in range(12):
        torch.cuda.synchronize()
        if where == "before":
            side_work(side)
        ev[0].record(stream)
        assert E.lib.esdp_backward_async(s.ctx, sp) == 0
        ev[1].record(stream)
        if where == "after":
            side_work(side)
        if where == "mid":
            time.sleep(0.001)
            side_work(side)
        torch.cuda.synchronize()
        if j >= 4:
            ts.append(ev[0].elapsed_time(ev[1]))
    return np.median(ts)

print(f"alone: backward {run('none', lo):.3f} ms")
for WHAT in ("kernel", "h2d_1KB", "h2d_4MB", "event"):
    for where in ("after", "mid"):
        print(f"side {WHAT:8s} {where:6s}: backward {run(where, lo):.3f} ms")
