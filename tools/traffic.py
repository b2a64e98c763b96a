"""DRAM traffic of one cfg2 backward pass (run under ncu with dram metrics; diagnostic):
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --cache-control none \
    -s <skip> -c <n> --csv --log-file out.csv python tools/traffic.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2511_15629_b200 as E
import workloads

s = E.Solver(workloads.cfg2(), keep_values=True)
for _ in range(3):
    s.backward()
torch.cuda.synchronize()
