import sys; sys.path.insert(0,'.')
import workloads, paper_2511_15629_b200 as E
inst=workloads.cfg2()
s=E.Solver(inst)
E.esdp_window_fallbacks(s.ctx)
s.backward()
n=E.esdp_window_fallbacks(s.ctx)
print("fallback rows", n, "of", inst.T*inst.K*inst.S)
