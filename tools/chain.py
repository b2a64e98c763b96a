"""Run the cfg2 backward a few times (for an ncu launch list of the chain's kernels): python tools/chain.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2511_15629_b200 as E
import workloads

s = E.Solver(workloads.cfg2(), keep_values=True)
for _ in range(3):
    s.backward()
torch.cuda.synchronize()
