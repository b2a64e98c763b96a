"""Warm per-launch kernel times and chain time per stage for the paper's Table 3 rows (rank-1; diagnostic)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2511_15629_b200 as E
import workloads

for hours, delta in ((4.0, 0.1), (100.0, 0.1), (4.0, 0.01), (100.0, 0.01)):
    inst = workloads.table3(hours=hours, delta=delta, T=512)
    s = E.Solver(inst, keep_values=False)
    for _ in range(3):
        s.backward()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(5):
        s.backward()
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t0) / 5 * 1e3
    print(f"table3 {hours:g}h delta {delta:g} (S={s.S}, A={s.A}, K={s.K}): {ms / inst.T * 1e3:.2f} us/stage | warm us/launch: "
          f"expectation {E.esdp_debug_time(s.ctx, 0):.2f} stencil {E.esdp_debug_time(s.ctx, 1):.2f} "
          f"empty {E.esdp_debug_time(s.ctx, 3):.2f}", flush=True)
    s.close()
