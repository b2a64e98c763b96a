"""Backward time per stage and warm per-launch kernel times (diagnostic):
python tools/stagetime.py cfg2|cfg4|cfg3ii|cfg2-rank1"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2511_15629_b200 as E
import workloads

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
if cfg == "cfg3ii":
    with E.Solver(workloads.cfg2(T=2, K=2)) as s0:
        inst = workloads.cfg3_gpu(s0.actions())
elif cfg == "cfg2-rank1":
    inst = workloads.cfg2(rank1=True)
else:
    inst = {"cfg2": workloads.cfg2, "cfg4": workloads.cfg4}[cfg]()
s = E.Solver(inst, keep_values=(cfg != "cfg4"))
for _ in range(3):
    s.backward()
torch.cuda.synchronize()
n = 10 if cfg != "cfg4" else 3
t0 = time.perf_counter()
for _ in range(n):
    s.backward()
torch.cuda.synchronize()
ms = (time.perf_counter() - t0) / n * 1e3
E.esdp_window_fallbacks(s.ctx)
E.esdp_window_level_tables(s.ctx)
s.backward()
print(f"{cfg} kind={s.stencil_kind}: backward {ms:.3f} ms ({ms / inst.T * 1e3:.2f} us/stage)"
      "  | warm us/launch: contract %.2f stencil %.2f" % (E.esdp_debug_time(s.ctx, 0), E.esdp_debug_time(s.ctx, 1)),
      "| per backward: fallback rows", E.esdp_window_fallbacks(s.ctx), "non-unimodal tables",
      E.esdp_window_level_tables(s.ctx), flush=True)
s.close()
