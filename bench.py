#!/usr/bin/env python
"""Benchmark of the B200 backward induction (arXiv 2511.15629) -- one JSON line on rank 0.

A step is one pass of the whole hot path over one synthetic instance:
  a2-a5  esdp backward induction (T-1 expectation contractions, T max-plus stencils, J) -- one CUDA graph
  a6     bid curves for every (t, i) at the median price state k = K/2 (T*S curves, the size of the
         paper's rank-1 bid set)
  a7     forward simulation of the argmax policy on --paths price paths
The metric is BASELINE.json's: DP cell-updates/s = T*S*K*A / step time (whole job over all ranks).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N > 1 is launched by torchrun.  --mode instances (default): every rank solves its own instance
(independent price draws, the cfg5-style instance sharding of SURVEY.md §8(e).3) with no data-path
collective -> "scaling": "weak".  --mode kpart: one instance, price-state rows split across ranks with an
NCCL all-gather of V_t every stage -> "scaling": "strong".
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

DMMA_PEAK_TFLOPS = 37.03  # FP64 tensor cores (mma.m8n8k4.f64), measured: profiles/r01_microbench.json
FP64_LANES_PER_SM = 64  # B200: 64 FP64 FMA lanes per SM (measured 62.8 DADD/SM/clk)


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f), "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "sm_max_mhz": 1965.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 20 ms.  Started before the warm-up (the tool
    needs ~0.1 s to start emitting); only the samples received between mark_begin() and mark_end() --
    the timed region -- are used, widened to the 3 nearest samples when the region is shorter than
    the sampling period (those fall in the adjacent warm-up / next step, the same load)."""

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
                                          "--format=csv,noheader,nounits", "-lms", "20"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except (OSError, FileNotFoundError):
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.perf_counter(), line.strip()))

    def wait_ready(self, extra_warmup, timeout=2.0):
        """Extra (untimed) warm-up steps until the sampler emits, so that it covers the timed region."""
        t = time.perf_counter()
        while self.proc is not None and not self.lines and time.perf_counter() - t < timeout:
            extra_warmup()

    def mark_begin(self):
        self.t0 = time.perf_counter()

    def mark_end(self):
        self.t1 = time.perf_counter()

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
        t0 = getattr(self, "t0", float("-inf"))
        t1 = getattr(self, "t1", float("inf"))
        inside = [x for x in self.lines if t0 <= x[0] <= t1 + 0.03]
        if len(inside) < 3 and self.lines:
            mid = 0.5 * (t0 + t1) if t0 > float("-inf") and t1 < float("inf") else self.lines[-1][0]
            inside = sorted(self.lines, key=lambda x: abs(x[0] - mid))[:3]
        for _, ln in inside:
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
    elif args.config == "cfg4":
        inst = workloads.cfg4()
    elif args.config == "table1":
        inst = workloads.table1_deterministic(0.01)
    elif args.config == "table3":
        inst = workloads.table3(hours=args.t3_hours, delta=args.t3_delta)
    elif args.config == "cfg3":
        import paper_2511_15629_b200 as E
        with E.Solver(workloads.cfg2(T=2, K=2)) as s:   # the Eq. 10 action grid of cfg2 (product's own)
            act = s.actions()
        inst = workloads.cfg3_gpu(act)
    else:
        raise SystemExit(f"unknown config {args.config}")
    if rank and args.config.startswith("cfg2"):
        # independent instance per rank (weak scaling): a different seeded jitter of the prices
        lam, _, _ = workloads.price_chain(inst.T, inst.K, 5.0 / 60.0, seed=workloads.SEED_BASE + 1000 + rank)
        inst.lam = lam
    return inst


# the paper's GPU rates (T*S*P*R / L40S time) for the Table 3 rows
T3_PAPER_RATE = {(4.0, 0.1): 8784 * 41 * 22 * 200 / 2.77, (20.0, 0.1): 8784 * 201 * 22 * 200 / 2.81,
                 (100.0, 0.1): 8784 * 1001 * 22 * 200 / 2.94, (4.0, 0.01): 8784 * 401 * 203 * 200 / 4.88,
                 (20.0, 0.01): 8784 * 2001 * 203 * 200 / 19.17, (100.0, 0.01): 8784 * 10001 * 203 * 200 / 86.67}

WORKLOAD = {
    "cfg2": "cfg2: ISO-NE-shaped 5-min RT day, Markov prices (T=288, S=1001, A=201, K=100, eta_c=eta_d=0.95)",
    "cfg2-rank1": "cfg2 with stagewise-independent prices (the paper's Alg. 1 case)",
    "cfg1": "cfg1b: T=24, S=101, A=21, K=5",
    "cfg4": "cfg4: full-year hourly horizon, per-stage P_t (T=8760, S=2001, A=401, K=200)",
    "table3": "the paper's Table 3 largest row (P:401): T=8784 hourly, S=10001 (100 h at delta=0.01), A=203, "
              "R=K=200 stagewise-independent price samples (rank-1); DP solve only, synthetic prices",
    "cfg3": "cfg3ii: cfg2 dimensions, prices shifted <= 0, non-concave payoff lambda p - 2|p| - 25 [p != 0]",
    "table1": "NEXT-3 Table-1 analog: deterministic (K=1) hourly year, T=8784, S=401, A=203 (delta=0.01)",
}


def run_ours(args):
    import ctypes

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
    kpart = args.mode == "kpart"
    # instances: every rank its own instance (weak scaling); kpart: one instance, K rows split (strong)
    inst = _instance(args, 0 if kpart else rank)
    dist_arg = None
    if kpart:
        nid = [E.esdp_nccl_unique_id() if rank == 0 else None]
        if world > 1:
            dist.broadcast_object_list(nid, src=0)
        dist_arg = (world, rank, nid[0])
    # table3 is the paper's Table 3 timing: the DP solve alone (no bid curves, no paths)
    solve_only = args.config == "table3"
    solver = E.Solver(inst, keep_values=not solve_only, dist=dist_arg,
                      force_brute=args.stencil == "brute", persist=args.plan == "persistent")
    T, S, A, K = solver.T, solver.S, solver.A, solver.K
    cells = T * S * K * A
    stream = torch.cuda.Stream(device=dev)
    sp = stream.cuda_stream

    # a6: bid-curve requests for every (t, i) at one of this rank's price states, device-resident
    k_lo, k_cnt, _ = E.esdp_partition(K, world if kpart else 1, rank if kpart else 0)
    kb = k_lo + k_cnt // 2
    tt, ii = np.meshgrid(np.arange(1, T + 1, dtype=np.int32), np.arange(S, dtype=np.int32), indexing="ij")
    req = np.stack([tt.ravel(), ii.ravel(), np.full(T * S, kb, np.int32)], 1).astype(np.int32)
    if (kpart and k_cnt == 0) or solve_only:
        req = req[:0]
    n_bid = req.shape[0]
    cap = A
    req_d = torch.from_numpy(req).to(dev)
    nv_d = torch.empty(max(n_bid, 1), dtype=torch.int32, device=dev)
    vert_d = torch.empty(max(n_bid, 1) * cap, dtype=torch.int16, device=dev)
    pr_d = torch.empty(max(n_bid, 1) * cap, dtype=torch.float64, device=dev)
    fused = args.bids == "fused" and n_bid > 0
    if fused:   # a6 inside the backward graph: stage t's curves in a side branch as soon as W_t exists
        E.esdp_set_bid_requests(solver.ctx, req, cap, nv_d.data_ptr(), vert_d.data_ptr(), None, pr_d.data_ptr())
    n_paths = args.paths // world if kpart else args.paths      # kpart: the paths are shared out too
    if solve_only:
        n_paths = 0
    per_d = torch.empty(max(n_paths, 1), dtype=torch.float64, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)  # > 126 MB L2
    ev = lambda: torch.cuda.Event(enable_timing=True)

    side = torch.cuda.Stream(device=dev)
    ev_bw, ev_bids = torch.cuda.Event(), torch.cuda.Event()
    with_sim = args.bids == "with-sim" and n_bid > 0

    def step(j, marks=None):
        if marks:
            marks[0].record(stream)
        E.esdp_backward_async(solver.ctx, sp)
        if marks:
            marks[1].record(stream)
        if with_sim:   # the bid curves on a side stream, concurrent with the (latency-bound) simulation
            ev_bw.record(stream)
            side.wait_event(ev_bw)
            E.esdp_bidcurves_dev(solver.ctx, n_bid, req_d.data_ptr(), cap, nv_d.data_ptr(), vert_d.data_ptr(),
                                 None, pr_d.data_ptr(), side.cuda_stream)
            ev_bids.record(side)
        elif n_bid and not fused:
            E.esdp_bidcurves_dev(solver.ctx, n_bid, req_d.data_ptr(), cap, nv_d.data_ptr(), vert_d.data_ptr(),
                                 None, pr_d.data_ptr(), sp)
        if marks:
            marks[2].record(stream)
        if n_paths:
            E.esdp_simulate_dev(solver.ctx, n_paths, 1234 + j + 7919 * rank, per_d.data_ptr(), sp)
        if with_sim:
            stream.wait_event(ev_bids)
        if marks:
            marks[3].record(stream)

    launches_per_step = E.esdp_launch_count(solver.ctx) + (1 if n_bid and not fused else 0) + 1
    clocks = ClockSampler(local)
    clocks.start()
    with torch.cuda.stream(stream):
        for j in range(args.warmup):
            flush.fill_(float(j))
            step(j)
        stream.synchronize()
        clocks.wait_ready(lambda: (flush.fill_(0.0), step(0), stream.synchronize()))
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)
        clocks.mark_begin()
        marks = [[ev() for _ in range(4)] for _ in range(args.steps)]
        part = np.zeros(3)
        phases = np.zeros(2)
        for j in range(args.steps):
            flush.fill_(float(j))          # L2 flush between timed steps (outside the events)
            step(j, marks[j])
            stream.synchronize()
            m = marks[j]
            part += [m[0].elapsed_time(m[1]), m[1].elapsed_time(m[2]), m[2].elapsed_time(m[3])]
        torch.cuda.synchronize(dev)
        clocks.mark_end()
        if world > 1:
            dist.barrier()
        clk = clocks.stop()
    J = E.esdp_objective(solver.ctx)
    sim_mean = float(per_d.mean().item()) if n_paths else None
    phases_ok = False
    if args.kernel_events and not kpart:
        # per-phase split from a separate context whose graph records CUDA events around the kernels of
        # ~16 sampled stages (kept out of the timed graph: event nodes break the PDL edges there); without
        # ESDP_KEEP_VALUES so that it fits next to the timed context
        try:
            with E.Solver(inst, keep_values=False, profile=True, force_brute=args.stencil == "brute",
                          persist=args.plan == "persistent") as prof:
                for j in range(args.warmup + args.steps):
                    prof.backward()
                    if j >= args.warmup:
                        phases += E.esdp_kernel_times(prof.ctx)
            phases_ok = True
        except E.EsdpError:
            pass
    part /= args.steps
    phases /= args.steps
    t_all = torch.tensor([part.sum()], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t_all, op=dist.ReduceOp.MAX)
    ms_step = float(t_all.item())
    units = cells * (1 if kpart else world)
    value = units / (ms_step * 1e-3)

    # --- end to end through the public API with host buffers (pinned), H2D/D2H inside the region
    lam_h = torch.from_numpy(np.ascontiguousarray(inst.lam)).pin_memory()
    P_h = torch.from_numpy(np.ascontiguousarray(inst.P)).pin_memory() if inst.P is not None else None
    pi_h = torch.from_numpy(np.ascontiguousarray(inst.pi)).pin_memory()
    h2d = lam_h.numel() * 8 + (P_h.numel() * 8 if P_h is not None else 0) + pi_h.numel() * 8
    dp = ctypes.POINTER(ctypes.c_double)
    as_p = lambda t: None if t is None else ctypes.cast(t.data_ptr(), dp)
    m_, v_ = ctypes.c_double(), ctypes.c_double()
    Jh = ctypes.c_double()
    # pipelined steps through the public API: step j launches its solve (with the fused bid curves), then
    # validates and enqueues the upload of step j+1's inputs into the other input slot (it overlaps solve
    # j), then enqueues the simulation and the D2H copies of J and the simulation statistics; step j's
    # results are read (event wait) after step j+1 has been launched.  Every step carries one full H2D of
    # inputs and one D2H of its results; the timed region starts with all earlier results read and ends
    # when the last step's results are on the host.
    load = lambda: E.lib.esdp_load_async(solver.ctx, as_p(lam_h), as_p(P_h), as_p(pi_h), None)
    J_h = torch.zeros(2, dtype=torch.float64).pin_memory()
    st_h = torch.zeros((2, 2), dtype=torch.float64).pin_memory()
    st_d = torch.zeros((2, 2), dtype=torch.float64, device=dev)
    done = [torch.cuda.Event(), torch.cuda.Event()]
    results = []
    assert load() == 0, E.esdp_last_error(solver.ctx)
    t0 = None

    def read(j):
        done[j % 2].synchronize()
        results.append((float(J_h[j % 2]), float(st_h[j % 2, 0]), float(st_h[j % 2, 1])))

    nstep = args.warmup + args.steps
    for j in range(nstep):
        if j == args.warmup:
            if j > 0:
                read(j - 1)
            torch.cuda.synchronize(dev)
            if world > 1:
                dist.barrier()
            t0 = time.perf_counter()
        assert E.lib.esdp_backward_async(solver.ctx, sp) == 0
        if n_bid and not fused:
            E.esdp_bidcurves_dev(solver.ctx, n_bid, req_d.data_ptr(), cap, nv_d.data_ptr(), vert_d.data_ptr(),
                                 None, pr_d.data_ptr(), sp)
        if j + 1 < nstep:
            st = load()                                    # the next step's inputs (validated, chunked H2D)
            assert st == 0, E.esdp_last_error(solver.ctx)
        assert E.lib.esdp_objective_async(solver.ctx, ctypes.c_void_p(J_h[j % 2:].data_ptr()), sp) == 0
        if n_paths:
            assert E.lib.esdp_simulate_async(solver.ctx, n_paths, 99 + j, ctypes.c_void_p(st_d[j % 2].data_ptr()),
                                             sp) == 0
            with torch.cuda.stream(stream):
                st_h[j % 2].copy_(st_d[j % 2], non_blocking=True)
        done[j % 2].record(stream)
        if j > 0 and j != args.warmup:
            read(j - 1)
    read(nstep - 1)
    e2e_times = [time.perf_counter() - t0]
    e2e_t = torch.tensor([sum(e2e_times)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(e2e_t, op=dist.ReduceOp.MAX)
    e2e_value = units / (float(e2e_t.item()) / args.steps)
    d2h = 8 + 16  # J, (mean, var)

    peaks, peak_kind = _peaks()
    sm_max = float(peaks.get("sm_max_mhz", 1965.0))
    n_sm = torch.cuda.get_device_properties(dev).multi_processor_count
    fp64_peak = n_sm * FP64_LANES_PER_SM * sm_max * 1e6 / 1e9          # G FP64 instr/s
    # algorithmic FP64 work of one backward on this rank: 2 per cell (add + max),
    # K FMA per (k, s) element of the expectation (T-1 stages); rows owned by this rank
    rows_here = k_cnt if kpart else K
    algo_ops = 2.0 * T * S * rows_here * A + (T - 1) * S * rows_here * (1 if inst.P is None else K) * 1.0
    bw_ms = part[0]
    achieved = algo_ops / (bw_ms * 1e-3) / 1e9
    hbm_bytes = 18.0 * T * rows_here * S                               # read W, write V + pol per (k, s, t)
    hbm_ach = hbm_bytes / (bw_ms * 1e-3) / 1e9
    plan = E.esdp_stencil_kind(solver.ctx)
    # DRAM traffic per backward from the committed ncu capture of this workload (cfg2, graph plan)
    traffic, traffic_note = None, None
    tr_path = os.path.join(ROOT, "profiles", "r01m_backward_traffic.json")
    if args.config == "cfg2" and not kpart and not (plan & 2) and os.path.exists(tr_path):
        with open(tr_path) as f:
            traffic = json.load(f)["per_backward_bytes"]
        traffic_note = ("dram__bytes_read.sum + dram__bytes_write.sum summed over one backward's kernels "
                        "(profiles/r01m_backward_traffic.json, ncu --cache-control none); algorithmic bytes "
                        "%.4g" % hbm_bytes)
    # the two stage kernels on their own (after the timed region): warm back-to-back launches of stage T-1's
    # kernel, CUDA events on the context's stream, each launch including its kernel boundary (no PDL)
    kernels = None
    if rank == 0 and not kpart and not (plan & 2) and T > 1:
        us_st = E.esdp_debug_time(solver.ctx, 1, 200)
        st_work = 2.0 * S * K * A
        kernels = {"stencil": {"kernel": "window_stencil_kernel" if plan & 1 else "stencil_kernel", "bound": "alu",
                               "us_per_launch": us_st, "work_per_launch": st_work,
                               "achieved": st_work / us_st / 1e3, "peak": fp64_peak, "unit": "G FP64 instr/s",
                               "frac": st_work / us_st / 1e3 / fp64_peak,
                               "note": "brute-force-equivalent FP64 instructions (2 per cell, SURVEY 8(d).3)",
                               "hbm": {"bytes_per_launch": 18.0 * S * K, "achieved": 18.0 * S * K / us_st / 1e3,
                                       "peak": float(peaks["hbm_gbs"]), "unit": "GB/s",
                                       "frac": 18.0 * S * K / us_st / 1e3 / float(peaks["hbm_gbs"]),
                                       "note": "read W_t, write V_t and the int16 policy per (k, s); W_t and V_t are "
                                               "L2-resident on cfg2, so DRAM sees little of it"}}}
        if inst.P is not None:
            us_ct = E.esdp_debug_time(solver.ctx, 0, 200)
            ct_flop = 2.0 * K * K * S
            kernels["expectation"] = {"kernel": "contract_dmma3_kernel" if K % 2 == 0 else "contract_dmma2_kernel",
                                      "bound": "tensor", "us_per_launch": us_ct, "work_per_launch": ct_flop,
                                      "achieved": ct_flop / us_ct / 1e6, "peak": DMMA_PEAK_TFLOPS, "unit": "TFLOP/s",
                                      "frac": ct_flop / us_ct / 1e6 / DMMA_PEAK_TFLOPS,
                                      "note": "FP64 DMMA; peak measured by tools/microbench/mb.cu "
                                              "(profiles/r01_microbench.json)"}
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
            "full_solve_s": part[0] / 1e3,
            "higher_is_better": True,
            "scaling": "strong" if kpart else "weak",
            # the paper's number for this exact workload shape: 41.2 G cell/s on an L40S
            "vs_baseline": (value / T3_PAPER_RATE[(args.t3_hours, args.t3_delta)]
                            if args.config == "table3" and (args.t3_hours, args.t3_delta) in T3_PAPER_RATE else None),
            "dtype": "f64",
            "data": ("synthetic (seeded ISO-NE-shaped hourly prices, R = 200 equally likely samples per hour, "
                     "DESIGN.md §4)" if args.config == "table3" else
                     "synthetic (seeded ISO-NE-shaped Markov price chain, DESIGN.md §4)"),
            "config": {"workload": WORKLOAD[args.config], "T": T, "S": S, "A": A, "K": K,
                       "bid_curves_per_step": n_bid, "sim_paths_per_step": n_paths,
                       "l2": "flushed between timed steps (256 MiB write outside the step events)",
                       "parallelism": (f"K-partitioned x{world} (NCCL all-gather of V_t per stage)" if kpart else
                                       f"instance-sharded x{world} (no data-path collective)" if world > 1 else "1 GPU"),
                       "plan": {"stencil": "window" if plan & 1 else "brute", "backward": "persistent" if plan & 2 else "graph",
                                "bidcurves": "fused into the backward graph" if fused else "after the backward"}},
            "gpu_launches": launches_per_step * args.steps,
            "ms_per_part": {"backward" + ("+bidcurves (fused branch)" if fused else ""): part[0],
                            "bidcurves": None if fused else part[1], "simulate": part[2]},
            "backward_phase_ms": ({"expectation": phases[0], "stencil": phases[1],
                                   "note": "separate profiled context (events around the kernels of ~16 stages)"}
                                  if phases_ok else None),
            "roofline": {"bound": "alu",
                         "kernel": "backward (%s)" % ("persistent dataflow kernel" if plan & 2 else "graph of 2T kernels"),
                         "achieved": achieved, "peak": fp64_peak, "unit": "G FP64 instr/s",
                         "frac": achieved / fp64_peak, "traffic": traffic, "traffic_note": traffic_note,
                         "peak_note": f"{n_sm} SMs x {FP64_LANES_PER_SM} FP64 lanes x {sm_max:.0f} MHz "
                                      f"(sm_max_mhz from MEASURED_PEAKS.json: {peak_kind})",
                         "work_per_launch": f"algorithmic FP64 instr: 2 per cell x T*S*K*A + K per (k,s) x (T-1)*S*K "
                                            f"= {algo_ops:.4g}"},
            "roofline_kernels": kernels,
            "roofline_hbm_literal": {"bound": "hbm", "achieved": hbm_ach, "peak": float(peaks["hbm_gbs"]),
                                     "unit": "GB/s", "frac": hbm_ach / float(peaks["hbm_gbs"]),
                                     "bytes_per_launch": hbm_bytes},
            "clocks": clk,
            "e2e": {"value": e2e_value, "unit": "cell-updates/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h},
            "J": J, "sim_mean_profit": sim_mean,
            "window_fallback_rows": E.esdp_window_fallbacks(solver.ctx),
        }
        if world == 1 and not args.no_cpu_baseline:
            out["cpu_baseline"] = cpu_baseline(inst, budget_s=args.cpu_budget)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    solver.close()
    return out


def run_sweep(args):
    """cfg5: a batch of storage configurations (different pbar, eta -> different action grids) over one
    price model, solved by one batch context (esdp_create_batch); each instance = backward + 1024
    simulated paths.  Ranks take disjoint instance ranges (weak scaling, no data-path collective)."""
    import numpy as np
    import torch
    import torch.distributed as dist
    import workloads
    import paper_2511_15629_b200 as E
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1 and not dist.is_initialized():
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    n = args.instances
    idx = [rank * n + j for j in range(n)]     # instance sharding across ranks (no communication)
    insts = workloads.cfg5_instances(idx)
    batch = E.Batch(insts, force_brute=args.stencil == "brute")   # one graph: one expectation + one stencil launch per stage
    stream = torch.cuda.Stream(device=dev)
    paths = 1024
    out_d = torch.empty(n * paths, dtype=torch.float64, device=dev)
    cells = sum(batch.T * batch.S * batch.K * a for a in batch.A)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    def step(j):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        batch.backward_async(stream.cuda_stream)
        batch.simulate_dev(paths, 17 + j, out_d.data_ptr(), stream.cuda_stream)
        e1.record(stream)
        return e0, e1

    clocks = ClockSampler(local)
    clocks.start()
    for j in range(args.warmup):
        step(j)
    torch.cuda.synchronize(dev)
    clocks.wait_ready(lambda: (step(0), stream.synchronize()))
    if world > 1:
        dist.barrier()
    clocks.mark_begin()
    ms = 0.0
    for j in range(args.steps):
        with torch.cuda.stream(stream):
            flush.fill_(float(j))              # L2 flush between timed steps (outside the events)
        e0, e1 = step(j)
        stream.synchronize()
        ms += e0.elapsed_time(e1)
    clocks.mark_end()
    clk = clocks.stop()
    ms /= args.steps
    t_all = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t_all, op=dist.ReduceOp.MAX)
    ms = float(t_all.item())
    # end to end: the per-instance storage parameters are host data that the batch is built from; the
    # shared price model is uploaded with it, and the J of every instance comes back
    J = batch.objective()
    As = list(batch.A)
    launches = (batch.launch_count() + 1) * args.steps
    batch.close()
    out = {"metric": "DP cell-updates/sec (T*S*K*A)", "value": cells * world / (ms * 1e-3), "unit": "cell-updates/s",
           "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic (cfg2 price chain; cfg5 storage sweep)",
           "config": {"workload": "cfg5 sweep sample: %d storage configurations per GPU in one batch context "
                                  "(pbar/delta in [10.42, 99], eta in [0.80, 0.99]; T=288, S=1001, K=100; A=%d..%d), "
                                  "1024 simulated paths each" % (n, min(As), max(As)),
                      "instances_per_gpu": n, "l2": "flushed between timed steps",
                      "plan": "esdp_create_batch: per stage one [K] x [n ld] expectation + one window launch"},
           "gpu_launches": launches, "J_mean": float(np.mean(J)),
           "clocks": clk}
    return out if rank == 0 else None


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
    ap.add_argument("--config", default="cfg2", choices=sorted(WORKLOAD) + ["cfg5"])
    ap.add_argument("--instances", type=int, default=16, help="cfg5: storage configurations per GPU")
    ap.add_argument("--t3-hours", type=float, default=100.0, help="table3: battery duration (hours)")
    ap.add_argument("--t3-delta", type=float, default=0.01, help="table3: SoC step (MWh)")
    ap.add_argument("--paths", type=int, default=65536)
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--ref-stages", type=int, default=24)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--kernel-events", type=int, default=1,
                    help="per-phase device timers inside the backward (persistent plan) / events (graph plan)")
    ap.add_argument("--bids", choices=["fused", "after", "with-sim"], default="fused",
                    help="bid curves as side branches of the backward graph (fused), one kernel after it, or one "
                         "kernel on a side stream concurrent with the simulation")
    ap.add_argument("--stencil", choices=["auto", "brute"], default="auto",
                    help="auto: exact sliding-window stencil where it applies; brute: every (i, a) cell")
    ap.add_argument("--plan", choices=["graph", "persistent"], default="graph",
                    help="backward as a CUDA graph of 2T kernels, or one persistent dataflow kernel (1 GPU)")
    ap.add_argument("--mode", choices=["instances", "kpart"], default="instances",
                    help="N>1: independent instances per rank (weak) or one K-partitioned instance (strong)")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        print("warning: --warmup < 3 violates the timing rules", file=sys.stderr)
    if args.impl == "reference":
        out = run_reference(args)
    elif args.config == "cfg5":
        out = run_sweep(args)
    else:
        out = run_ours(args)
    if out is not None:
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
