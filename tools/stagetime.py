"""Backward time per stage and warm per-launch kernel times, fused stage kernel vs the two-kernel stage
(diagnostic): ESDP_FUSED=0|1 python tools/fusedtime.py cfg2|cfg4|cfg3ii"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2511_15629_b200 as E
import workloads

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
if cfg == "cfg3ii":
    with E.Solver(workloads.cfg2(T=2, K=2)) as s0:
        inst = workloads.cfg3_gpu(s0.actions())
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
kind = s.stencil_kind
line = f"{cfg} fused={os.environ.get('ESDP_FUSED', '1')} kind={kind}: backward {ms:.3f} ms ({ms / inst.T * 1e3:.2f} us/stage)"
if kind & 4:
    line += "  | warm us/launch: stage %.2f" % E.esdp_debug_time(s.ctx, 4)
else:
    line += "  | warm us/launch: contract %.2f stencil %.2f" % (E.esdp_debug_time(s.ctx, 0), E.esdp_debug_time(s.ctx, 1))
print(line, "fallbacks", E.esdp_window_fallbacks(s.ctx), "level/nonuni tables", E.esdp_window_level_tables(s.ctx), flush=True)
s.close()
