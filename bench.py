#!/usr/bin/env python
"""Benchmark of the B200 backward induction (arXiv 2511.15629) -- one JSON line on rank 0.

A step is one pass of the whole hot path over one synthetic instance:
  a2-a5  esdp backward induction (T-1 expectation contractions, T max-plus stencils, J) -- one CUDA graph
  a6     bid curves for every (t, i) at the median price state k = K/2 (T*S curves, the size of the
         paper's rank-1 bid set)
  a7     forward simulation of the argmax policy on --paths price paths
The metric is BASELINE.json's: DP cell-updates/s = T*S*K*A / step time (whole job over all ranks).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N > 1 is launched by torchrun: every rank solves its own instance (independent price draws, the
cfg5-style instance sharding of SURVEY.md §8(e).3) with no data-path collective -> "scaling": "weak".
--impl reference times the FP64 CPU oracle (oracle/) on this host's cores on a bounded sample of the
same workload (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

FP64_LANES_PER_SM = 64  # B200: 64 FP64 FMA lanes per SM (measured 62.8 DADD/SM/clk)


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f), "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "sm_max_mhz": 1965.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.dev = device_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except (OSError, FileNotFoundError):
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax = float(f[2])
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


def _instance(args, rank):
    import workloads
    if args.config == "cfg2":
        inst = workloads.cfg2()
    elif args.config == "cfg2-rank1":
        inst = workloads.cfg2(rank1=True)
    elif args.config == "cfg1":
        inst = workloads.cfg1("b")
    else:
        raise SystemExit(f"unknown config {args.config}")
    if rank:
        # independent instance per rank (weak scaling): a different seeded jitter of the prices
        lam, _, _ = workloads.price_chain(inst.T, inst.K, 5.0 / 60.0, seed=workloads.SEED_BASE + 1000 + rank)
        inst.lam = lam
    return inst


WORKLOAD = {
    "cfg2": "cfg2: ISO-NE-shaped 5-min RT day, Markov prices (T=288, S=1001, A=201, K=100, eta_c=eta_d=0.95)",
    "cfg2-rank1": "cfg2 with stagewise-independent prices (the paper's Alg. 1 case)",
    "cfg1": "cfg1b: T=24, S=101, A=21, K=5",
}


def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2511_15629_b200 as E

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    inst = _instance(args, rank)
    solver = E.Solver(inst, keep_values=True, profile=args.kernel_events)
    T, S, A, K = solver.T, solver.S, solver.A, solver.K
    cells = T * S * K * A
    stream = torch.cuda.Stream(device=dev)
    sp = stream.cuda_stream

    # a6: bid-curve requests for every (t, i) at k = K/2, device-resident
    kb = K // 2
    tt, ii = np.meshgrid(np.arange(1, T + 1, dtype=np.int32), np.arange(S, dtype=np.int32), indexing="ij")
    req = np.stack([tt.ravel(), ii.ravel(), np.full(T * S, kb, np.int32)], 1).astype(np.int32)
    n_bid = req.shape[0]
    cap = A
    req_d = torch.from_numpy(req).to(dev)
    nv_d = torch.empty(n_bid, dtype=torch.int32, device=dev)
    vert_d = torch.empty(n_bid * cap, dtype=torch.int16, device=dev)
    pr_d = torch.empty(n_bid * cap, dtype=torch.float64, device=dev)
    per_d = torch.empty(args.paths, dtype=torch.float64, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)  # > 126 MB L2

    def step(j):
        E.esdp_backward_async(solver.ctx, sp)
        E.esdp_bidcurves_dev(solver.ctx, n_bid, req_d.data_ptr(), cap, nv_d.data_ptr(), vert_d.data_ptr(),
                             None, pr_d.data_ptr(), sp)
        E.esdp_simulate_dev(solver.ctx, args.paths, 1234 + j, per_d.data_ptr(), sp)

    launches_per_step = E.esdp_launch_count(solver.ctx) + 2
    with torch.cuda.stream(stream):
        for j in range(args.warmup):
            flush.fill_(float(j))
            step(j)
        stream.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)
        clocks = ClockSampler(local)
        clocks.start()
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        tot_ms, con_ms, sten_ms = 0.0, 0.0, 0.0
        for j in range(args.steps):
            flush.fill_(float(j))          # L2 flush between timed steps (outside the events)
            evs[j][0].record(stream)
            step(j)
            evs[j][1].record(stream)
            stream.synchronize()
            if args.kernel_events:
                c_ms, s_ms = E.esdp_kernel_times(solver.ctx)   # per launch, sampled stages
                con_ms += c_ms * (T - 1)
                sten_ms += s_ms * T
            tot_ms += evs[j][0].elapsed_time(evs[j][1])
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        clk = clocks.stop()
    J = E.esdp_objective(solver.ctx)
    sim_mean = float(per_d.mean().item())
    t_all = torch.tensor([tot_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t_all, op=dist.ReduceOp.MAX)
    ms_step = float(t_all.item()) / args.steps
    value = cells * world / (ms_step * 1e-3)

    # --- end to end through the public API with host buffers (pinned), H2D/D2H inside the region
    lam_h = torch.from_numpy(np.ascontiguousarray(inst.lam)).pin_memory()
    P_h = torch.from_numpy(np.ascontiguousarray(inst.P)).pin_memory() if inst.P is not None else None
    pi_h = torch.from_numpy(np.ascontiguousarray(inst.pi)).pin_memory()
    h2d = lam_h.numel() * 8 + (P_h.numel() * 8 if P_h is not None else 0) + pi_h.numel() * 8
    import ctypes
    dp = ctypes.POINTER(ctypes.c_double)
    as_p = lambda t: None if t is None else ctypes.cast(t.data_ptr(), dp)
    m, v = ctypes.c_double(), ctypes.c_double()
    Jh = ctypes.c_double()
    e2e_times = []
    for j in range(args.warmup + args.steps):
        if world > 1 and j == args.warmup:
            dist.barrier()
        t0 = time.perf_counter()
        st = E.lib.esdp_load(solver.ctx, as_p(lam_h), as_p(P_h), as_p(pi_h), None)
        assert st == 0, E.esdp_last_error(solver.ctx)
        assert E.lib.esdp_backward(solver.ctx, sp, ctypes.byref(Jh)) == 0
        E.esdp_bidcurves_dev(solver.ctx, n_bid, req_d.data_ptr(), cap, nv_d.data_ptr(), vert_d.data_ptr(),
                             None, pr_d.data_ptr(), sp)
        assert E.lib.esdp_simulate(solver.ctx, args.paths, 99 + j, ctypes.byref(m), ctypes.byref(v), None) == 0
        t1 = time.perf_counter()
        if j >= args.warmup:
            e2e_times.append(t1 - t0)
    e2e_t = torch.tensor([sum(e2e_times)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(e2e_t, op=dist.ReduceOp.MAX)
    e2e_value = cells * world / (float(e2e_t.item()) / args.steps)
    d2h = 8 + 16  # J, (mean, var)

    peaks, peak_kind = _peaks()
    sm_max = float(peaks.get("sm_max_mhz", 1965.0))
    n_sm = torch.cuda.get_device_properties(dev).multi_processor_count
    fp64_peak = n_sm * FP64_LANES_PER_SM * sm_max * 1e6 / 1e9          # Gop/s
    st_launch_ms = max(sten_ms, 1e-9) / (args.steps * T)
    ops_per_launch = 2.0 * K * S * A                                    # 1 DADD + 1 compare per cell
    achieved = ops_per_launch / (st_launch_ms * 1e-3) / 1e9
    hbm_bytes_launch = 18.0 * K * S                                     # read W 8 B, write V 8 B + pol 2 B
    hbm_ach = hbm_bytes_launch / (st_launch_ms * 1e-3) / 1e9
    out = None
    if rank == 0:
        out = {
            "metric": "DP cell-updates/sec (T*S*K*A)",
            "value": value,
            "unit": "cell-updates/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": ms_step,
            "full_solve_s": ms_step / 1e3,
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "f64",
            "data": "synthetic (seeded ISO-NE-shaped Markov price chain, DESIGN.md §4)",
            "config": {"workload": WORKLOAD[args.config], "T": T, "S": S, "A": A, "K": K,
                       "bid_curves_per_step": n_bid, "sim_paths_per_step": args.paths,
                       "l2": "flushed between timed steps (256 MiB write outside the step events)",
                       "parallelism": f"instance-sharded x{world} (no data-path collective)" if world > 1 else "1 GPU"},
            "gpu_launches": launches_per_step * args.steps,
            "kernel_ms_per_step": {"stencil": sten_ms / args.steps, "contract": con_ms / args.steps,
                                   "other": ms_step - (sten_ms + con_ms) / args.steps},
            "roofline": {"bound": "alu", "kernel": "stencil_kernel (max-plus + argmax, FP64 pipe)",
                         "achieved": achieved, "peak": fp64_peak, "unit": "FP64 Gop/s",
                         "frac": achieved / fp64_peak, "traffic": None,
                         "peak_note": f"{n_sm} SMs x {FP64_LANES_PER_SM} FP64 lanes x {sm_max:.0f} MHz "
                                      f"(sm_max_mhz from MEASURED_PEAKS.json: {peak_kind})",
                         "work_per_launch": f"2 FP64 ops x K*S*A = {ops_per_launch:.4g}"},
            "roofline_hbm_literal": {"bound": "hbm", "achieved": hbm_ach, "peak": float(peaks["hbm_gbs"]),
                                     "unit": "GB/s", "frac": hbm_ach / float(peaks["hbm_gbs"]),
                                     "bytes_per_launch": hbm_bytes_launch},
            "clocks": clk,
            "e2e": {"value": e2e_value, "unit": "cell-updates/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h},
            "J": J, "sim_mean_profit": sim_mean,
        }
        if world == 1 and not args.no_cpu_baseline:
            out["cpu_baseline"] = cpu_baseline(inst, budget_s=args.cpu_budget)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    solver.close()
    return out


def cpu_baseline(inst, budget_s=20.0, n_stages=None):
    """The FP64 oracle as it stands, on this host's cores, on a bounded sample of the same workload:
    the last n stages of the backward pass (t = T .. T-n+1, every (k, i) row)."""
    import oracle
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from helpers import to_oracle
    pr = to_oracle(inst)
    S, A = oracle.dims(pr)
    cores = os.cpu_count() or 1
    if n_stages is None:
        t0 = time.perf_counter()
        oracle.backward(pr, t_stop=inst.T - 1, nthreads=cores)   # 2 stages to size the sample
        dt = max(time.perf_counter() - t0, 1e-3) / 2
        n_stages = int(max(2, min(inst.T, budget_s / dt)))
    t0 = time.perf_counter()
    oracle.backward(pr, t_stop=inst.T - n_stages + 1, nthreads=cores)
    dt = time.perf_counter() - t0
    cells = n_stages * S * inst.K * A
    return {"value": cells / dt, "unit": "cell-updates/s", "cores": cores, "kind": "oracle",
            "sample": f"oracle backward, last {n_stages} of {inst.T} stages of the same instance "
                      f"(all K*S rows, OpenMP {cores} threads), {dt:.2f} s"}


def run_reference(args):
    """--impl reference: the oracle, timed on the host cores; each step is a bounded sample."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return None
    import oracle
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from helpers import to_oracle
    inst = _instance(args, 0)
    pr = to_oracle(inst)
    S, A = oracle.dims(pr)
    cores = os.cpu_count() or 1
    n_stages = max(2, min(inst.T, args.ref_stages))
    cells = n_stages * S * inst.K * A
    for _ in range(args.warmup):
        oracle.backward(pr, t_stop=inst.T - n_stages + 1, nthreads=cores)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        oracle.backward(pr, t_stop=inst.T - n_stages + 1, nthreads=cores)
        times.append(time.perf_counter() - t0)
    ms = 1e3 * sum(times) / len(times)
    value = cells / (ms * 1e-3)
    sample = f"oracle backward, last {n_stages} of {inst.T} stages per step (all K*S rows, {cores} threads)"
    return {"impl": "reference", "metric": "DP cell-updates/sec (T*S*K*A)", "value": value,
            "unit": "cell-updates/s", "n_gpus": int(os.environ.get("WORLD_SIZE", "1")), "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": WORKLOAD[args.config], "sample": sample},
            "cpu_baseline": {"value": value, "unit": "cell-updates/s", "cores": cores, "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": value, "unit": "cell-updates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="cfg2", choices=sorted(WORKLOAD))
    ap.add_argument("--paths", type=int, default=65536)
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--ref-stages", type=int, default=24)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--kernel-events", type=int, default=1,
                    help="CUDA events around the kernels of ~16 sampled stages per step (live launch durations)")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        print("warning: --warmup < 3 violates the timing rules", file=sys.stderr)
    out = run_reference(args) if args.impl == "reference" else run_ours(args)
    if out is not None:
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
