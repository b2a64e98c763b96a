"""Window vs brute-force stencil warm launch time across action counts (cfg5 instances)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_15629_b200 as E
import workloads

for j in (0, 100, 200, 300, 400, 500, 600, 700, 800, 900, 1000):
    inst = workloads.cfg5_instances([j], T=8, K=100)[0]
    s = E.Solver(inst, keep_values=True)
    s.backward()
    w = E.esdp_debug_time(s.ctx, 1)
    b = E.esdp_debug_time(s.ctx, 2)
    print(f"A={s.A:4d} window={'y' if s.stencil_kind & 1 else 'n'} ctx-stencil {w:6.2f} us  brute {b:6.2f} us")
    s.close()
