"""Warm per-kernel launch times and backward-graph time on cfg2 (diagnostic): python tools/ktime.py"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2511_15629_b200 as E
import workloads

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
inst = workloads.cfg2() if cfg == "cfg2" else workloads.cfg2(rank1=True)


def bw_time(s, n=10):
    for _ in range(3):
        s.backward()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        s.backward()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n * 1e3


for keep in (True,):
    for brute in (False,):
        for pdl, dmma in ((True, True), (False, True), (True, "l2"), (True, False)):
            if dmma == "l2":
                import types
                s = E.Solver.__new__(E.Solver)
                s.ctx = E.esdp_create(inst.T, inst.K, inst.pbar, inst.sbar, inst.s0, inst.eta_c, inst.eta_d, inst.delta,
                                      inst.lam, inst.P, inst.pi, None, 0, None,
                                      (E.ESDP_KEEP_VALUES if keep else 0) | (E.ESDP_FORCE_BRUTE if brute else 0) | E.ESDP_DMMA_L2)
                s.T, s.S, s.A, s.K = E.esdp_dims(s.ctx)
                s.stencil_kind = E.esdp_stencil_kind(s.ctx)
            else:
                s = E.Solver(inst, keep_values=keep, force_brute=brute, pdl=pdl, dmma=dmma)
            ms = bw_time(s)
            line = f"keep={int(keep)} stencil={'brute ' if not s.stencil_kind else 'window'} pdl={int(pdl)} dmma={dmma}: backward {ms:.3f} ms ({ms / inst.T * 1e3:.2f} us/stage)"
            if keep and pdl:
                line += "  | warm us/launch: contract %.2f stencil %.2f objective %.2f" % (
                    E.esdp_debug_time(s.ctx, 0), E.esdp_debug_time(s.ctx, 1), E.esdp_debug_time(s.ctx, 3))
            print(line, flush=True)
            s.close()

s = E.Solver(inst, keep_values=True, force_brute=False)
ms = bw_time(s)
print(f"graph keep=1: backward {ms:.3f} ms ({ms / inst.T * 1e3:.2f} us/stage)", flush=True)
s.close()
