"""cfg5 batch backward, a few passes (for ncu captures of the batch kernels): python tools/batchrun.py [n] [ozaki]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
# one chain over the whole batch: the captured launches then pair with bench.py's full-batch launch timing
# (esdp_batch_kernel_time) in the roofline fields
os.environ.setdefault("ESDP_BATCH_GROUPS", "1")
import torch
import paper_2511_15629_b200 as E
import workloads

n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
idx = [(j * 1024) // n for j in range(n)]
oz = len(sys.argv) > 2 and sys.argv[2] == "ozaki"
with E.Batch(workloads.cfg5_instances(idx), ozaki=oz) as b:
    for _ in range(2):
        b.backward()
    torch.cuda.synchronize()
    print("batch", n, "plan", b.plan, "A mean", sum(b.A) / n, "window us/launch %.1f expectation us/launch %.1f" % (b.kernel_time(1, 20), b.kernel_time(0, 20)))
