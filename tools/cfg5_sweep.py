"""The whole cfg5 sweep (1024 storage configurations: 32 durations x 32 efficiencies, T=288, S=1001, K=100) on
ONE GPU, in the 8 stratified shards of 128 configurations that `bench.py --config cfg5 --gpus 8` gives its 8
ranks (rank r: configurations r, r + 8, r + 16, ...), one batch context per shard, backward + 1024 simulated
paths per configuration.  Reports the time per shard and for the sweep, and checks J of a sample of
configurations (two per shard) bit for bit against the FP64 oracle: python tools/cfg5_sweep.py"""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import torch
import paper_2511_15629_b200 as E
import workloads
import oracle
from helpers import to_oracle

world, n = 8, 128
covered = []
total = 0.0
Js = {}
for r in range(world):
    idx = [((r + world * j) * 1024) // (world * n) for j in range(n)]
    covered += idx
    insts = workloads.cfg5_instances(idx)
    out = torch.empty(n * 1024, dtype=torch.float64, device="cuda")
    st = torch.cuda.Stream()
    with E.Batch(insts) as b:
        b.backward(); torch.cuda.synchronize()             # warm
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        b.backward_async(st.cuda_stream)
        b.simulate_dev(1024, 17, out.data_ptr(), st.cuda_stream)
        e1.record(st)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        total += ms
        J = b.objective()
        for j in (0, n - 1):
            Js[idx[j]] = (J[j], insts[j])
    print(f"shard {r}: configurations {idx[0]}..{idx[-1]} (every {world}), {ms:.1f} ms", flush=True)
assert sorted(covered) == list(range(1024)), "the shards cover the sweep exactly once"
print(f"sweep: 1024 configurations in {total:.1f} ms on one GPU ({total / world:.1f} ms per shard = per rank on 8 GPUs)")
bad = 0
for m, (Jg, inst) in sorted(Js.items()):
    ref = oracle.backward(to_oracle(inst), nthreads=os.cpu_count() or 1)
    bad += Jg != ref.J
    print(f"configuration {m}: J = {Jg:.6f} {'==' if Jg == ref.J else '!='} oracle {ref.J:.6f}", flush=True)
print("J bit-identical on the sample" if bad == 0 else f"{bad} mismatches")
