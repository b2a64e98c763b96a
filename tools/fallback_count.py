import sys; sys.path.insert(0, '/root/repo')
import paper_2511_15629_b200 as E, workloads
for name, inst in [("cfg2", workloads.cfg2()), ("t3big", workloads.table3(hours=100.0, delta=0.01, T=64))]:
    s = E.Solver(inst, keep_values=True)
    E.esdp_window_fallbacks(s.ctx)
    s.backward()
    print(name, "fallback rows per backward", E.esdp_window_fallbacks(s.ctx), "of", inst.T * s.S * s.K)
    s.close()
