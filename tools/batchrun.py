"""cfg5 batch backward, a few passes (for ncu captures of the batch kernels): python tools/batchrun.py [n]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2511_15629_b200 as E
import workloads

n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
idx = [(j * 1024) // n for j in range(n)]
with E.Batch(workloads.cfg5_instances(idx)) as b:
    for _ in range(2):
        b.backward()
    torch.cuda.synchronize()
    print("batch", n, "A mean", sum(b.A) / n, "window us/launch %.1f expectation us/launch %.1f" % (b.kernel_time(1, 20), b.kernel_time(0, 20)))
