#!/usr/bin/env python
"""Benchmark of the B200 backward induction (arXiv 2511.15629) -- one JSON line on rank 0.

A step is one pass of the whole hot path over one synthetic instance:
  a2-a5  esdp backward induction (T-1 expectation contractions, T max-plus stencils, J) -- one CUDA graph
  a6     bid curves for every (t, i) at the median price state k = K/2 (T*S curves, the size of the
         paper's rank-1 bid set)
  a7     forward simulation of the argmax policy on --paths price paths
The metric is BASELINE.json's: DP cell-updates/s = T*S*K*A / step time (whole job over all ranks).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N > 1: launched by torchrun (one process per GPU), or self-launched through torch.distributed.run when
--gpus N > 1 and WORLD_SIZE is unset.  The main line is --mode kpart (default for N > 1): one instance,
price-state rows split across ranks with an NCCL all-gather of V_t every stage ->
"scaling": "strong"; rank 0 then checks J, V_1 and every policy stage bit-equal to a 1-GPU context
("parity_vs_1gpu").  The instance-sharded run (every rank its own instance, no
data-path collective) is measured after it and reported under "instances_weak".
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


def _workload_name(args):
    if args.config == "table3" and (args.t3_hours, args.t3_delta) != (100.0, 0.01):
        return ("the paper's Table 3 row (P:395-401) of a %g h battery at delta=%g: T=8784 hourly, R=K=200 "
                "stagewise-independent price samples (rank-1); DP solve only, synthetic prices"
                % (args.t3_hours, args.t3_delta))
    return WORKLOAD[args.config]


def run_ours(args, mode):
    import ctypes

    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2511_15629_b200 as E

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    kpart = mode == "kpart"
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
    solver = E.Solver(inst, keep_values=not solve_only, dist=dist_arg, force_brute=args.stencil == "brute")
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
            with E.Solver(inst, keep_values=False, profile=True, force_brute=args.stencil == "brute") as prof:
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
    hbm_peak = float(peaks["hbm_gbs"])
    sm_max = float(peaks.get("sm_max_mhz", 1965.0))
    n_sm = torch.cuda.get_device_properties(dev).multi_processor_count
    fp64_peak = n_sm * FP64_LANES_PER_SM * sm_max * 1e6          # FP64 thread-instructions/s (DFMA/DADD lanes)
    rows_here = k_cnt if kpart else K
    plan = E.esdp_stencil_kind(solver.ctx)
    kprof = _kernel_profile(args.config) if not kpart and args.stencil == "auto" else None
    kernels, binding, bw_only_ms = None, None, None
    if rank == 0 and world == 1 and T > 1 and rows_here > 0:
        # the two stage kernels on their own (after the timed region): warm back-to-back launches of stage
        # T-1's kernel, CUDA events on the context's stream, each launch including its kernel boundary
        us_st = E.esdp_debug_time(solver.ctx, 1, 200)
        outs = S * rows_here
        st_bytes = 18.0 * outs                # read W_t (8 B), write V_t (8 B) and pol_t (2 B) per output (k, s)
        win = {"kernel": "window_stencil_kernel" if plan & 1 else "stencil_kernel", "bound": "hbm",
               "us_per_launch": us_st, "bytes_per_launch": st_bytes, "achieved": st_bytes / us_st / 1e3,
               "peak": hbm_peak, "unit": "GB/s", "frac": st_bytes / us_st / 1e3 / hbm_peak,
               "traffic": None, "instr_per_output": None}
        if kprof and "window" in kprof:
            win["traffic"] = kprof["window"]["dram_bytes_per_launch"]
            win["instr_per_output"] = kprof["window"]["warp_inst_per_launch"] * 32.0 / outs
            win["fp64_thread_inst_per_launch"] = kprof["window"]["fp64_thread_inst_per_launch"]
        kernels = {"stencil": win}
        if inst.P is not None:
            us_ct = E.esdp_debug_time(solver.ctx, 0, 200)
            ct_flop = 2.0 * K * rows_here * S
            kernels["expectation"] = {"kernel": "contract_dmma3_kernel" if (plan & 2 and K % 2 == 0) else "contract_dmma2/dfma",
                                      "bound": "tensor", "us_per_launch": us_ct, "flop_per_launch": ct_flop,
                                      "achieved": ct_flop / us_ct / 1e6, "peak": DMMA_PEAK_TFLOPS, "unit": "TFLOP/s",
                                      "frac": ct_flop / us_ct / 1e6 / DMMA_PEAK_TFLOPS,
                                      "note": "FP64 DMMA (mma.m8n8k4.f64); peak measured by tools/microbench/mb.cu "
                                              "(profiles/r01_microbench.json)"}
        us_dep = E.esdp_debug_time(solver.ctx, 3, 200)   # a 1-block dependent kernel: the cost of a boundary
        # the backward alone (no bid curves, no paths), events around 10 solves of a plain context
        with E.Solver(inst, keep_values=False, force_brute=args.stencil == "brute") as plain:
            e0, e1 = ev(), ev()
            ps = torch.cuda.Stream(device=dev)
            for _ in range(3):
                E.esdp_backward_async(plain.ctx, ps.cuda_stream)
            e0.record(ps)
            for _ in range(10):
                E.esdp_backward_async(plain.ctx, ps.cuda_stream)
            e1.record(ps)
            torch.cuda.synchronize(dev)
            bw_only_ms = e0.elapsed_time(e1) / 10
        # binding roofline of the backward: the slowest of HBM (algorithmic bytes),
        # compute (FP64 instructions the stencil actually executes, from ncu, + the DMMA flops) and the
        # dependent-launch floor (2 kernel boundaries per stage), over the measured backward time
        algo_bytes = 18.0 * T * S * rows_here + (8.0 * (T - 1) * K * rows_here if inst.P is not None else 0.0)
        t_hbm = algo_bytes / (hbm_peak * 1e9) * 1e3
        t_dmma = (T - 1) * 2.0 * K * rows_here * S / (DMMA_PEAK_TFLOPS * 1e12) * 1e3 if inst.P is not None else 0.0
        t_fp64 = (T * win["fp64_thread_inst_per_launch"] / fp64_peak * 1e3) if "fp64_thread_inst_per_launch" in win else None
        t_comp = None if t_fp64 is None else t_fp64 + t_dmma
        t_sync = T * (2 if inst.P is not None else 1) * us_dep * 1e-3
        cands = {"hbm": t_hbm, "compute": t_comp, "launch": t_sync}
        bind = max((k for k in cands if cands[k] is not None), key=lambda k: cands[k])
        binding = {"t_hbm_ms": t_hbm, "t_compute_ms": t_comp, "t_fp64_stencil_ms": t_fp64, "t_dmma_ms": t_dmma,
                   "t_launch_floor_ms": t_sync, "us_per_dependent_launch": us_dep, "t_backward_ms": bw_only_ms,
                   "binding": bind, "frac": cands[bind] / bw_only_ms,
                   "note": "max(t_HBM, t_compute, T x boundaries) / measured backward (SURVEY 8(d).3(iii)); "
                           "t_compute from the FP64 instructions the stencil executes (ncu, profiles/) plus the "
                           "DMMA flops at the measured DMMA peak; algorithmic bytes %.4g per backward" % algo_bytes}
    out = None
    if rank == 0:
        roof = None
        if kernels:
            w = kernels["stencil"]
            roof = {"bound": "hbm", "achieved": w["achieved"], "peak": hbm_peak, "unit": "GB/s", "frac": w["frac"],
                    "traffic": w["traffic"], "kernel": w["kernel"], "us_per_launch": w["us_per_launch"],
                    "bytes_per_launch": w["bytes_per_launch"], "instr_per_output": w["instr_per_output"],
                    "work_per_launch": "18 B per output (k, s): read W_t, write V_t (FP64) and pol_t (int16); "
                                       "S*K outputs = %d" % (S * rows_here),
                    "peak_note": "MEASURED_PEAKS.json hbm_gbs (%s)" % peak_kind,
                    "note": "the dominant kernel of the step (ncu launch list, profiles/); warm launches timed "
                            "with CUDA events after the timed region; V_t / W_t of a single cfg2 instance stay "
                            "L2-resident, so this kernel is latency- and issue-bound, not DRAM-bound "
                            "(roofline_binding)"}
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
            "config": {"workload": _workload_name(args), "T": T, "S": S, "A": A, "K": K,
                       "bid_curves_per_step": n_bid, "sim_paths_per_step": n_paths,
                       "l2": "flushed between timed steps (256 MiB write outside the step events)",
                       "parallelism": (f"K-partitioned x{world} (NCCL all-gather of V_t per stage)" if kpart else
                                       f"instance-sharded x{world} (no data-path collective)" if world > 1 else "1 GPU"),
                       "plan": {"stencil": "window" if plan & 1 else "brute",
                                "expectation": "FP64 DMMA" if plan & 2 else "DFMA",
                                "bidcurves": "fused into the backward graph" if fused else "after the backward"}},
            "gpu_launches": launches_per_step * args.steps,
            "ms_per_part": {"backward" + ("+bidcurves (fused branch)" if fused else ""): part[0],
                            "bidcurves": None if fused else part[1], "simulate": part[2],
                            "backward_only": bw_only_ms},
            "backward_phase_ms": ({"expectation": phases[0], "stencil": phases[1],
                                   "note": "separate profiled context (events around the kernels of ~16 stages)"}
                                  if phases_ok else None),
            "roofline": roof,
            "roofline_binding": binding,
            "roofline_kernels": kernels,
            "clocks": clk,
            "e2e": {"value": e2e_value, "unit": "cell-updates/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h},
            "J": J, "sim_mean_profit": sim_mean,
            "window_fallback_rows": E.esdp_window_fallbacks(solver.ctx),
        }
        if kprof and "window" in kprof and roof is not None:
            _issue_frac(roof, kprof["window"]["warp_inst_per_launch"], clk, dev)
        if world == 1 and not args.no_cpu_baseline:
            out["cpu_baseline"] = cpu_baseline(inst, budget_s=args.cpu_budget)
    if kpart and world > 1:
        out_p = _parity_vs_1gpu(E, solver, inst, rank, world, dev)
        if rank == 0:
            out.update(out_p)
    solver.close()
    return out


def _parity_vs_1gpu(E, solver, inst, rank, world, dev):
    """K-partitioned run vs one GPU (an all-gather is a copy): rank 0 solves the same instance
    on a context of its own and compares J, V_1 and every stage's policy bit for bit; every rank reports its
    communicator's rank count."""
    import numpy as np
    import torch
    import torch.distributed as dist
    w, r, nr = E.esdp_dist_info(solver.ctx)
    ok_local = torch.tensor([1 if (w == world and r == rank and nr == world) else 0], device=dev)
    dist.all_reduce(ok_local, op=dist.ReduceOp.MIN)
    res = {}
    if rank == 0:
        J = E.esdp_objective(solver.ctx)
        V1 = E.esdp_values(solver.ctx, 1, want_W=False)
        pols = [E.esdp_policy(solver.ctx, t) for t in range(1, solver.T + 1)]
        with E.Solver(inst, keep_values=False) as one:
            J1 = one.backward()
            same = (J == J1 and np.array_equal(V1, E.esdp_values(one.ctx, 1, want_W=False)) and
                    all(np.array_equal(pols[t - 1], one.policy(t)) for t in range(1, solver.T + 1)))
        res = {"parity_vs_1gpu": bool(same), "comm_nranks_ok": bool(ok_local.item()), "J_1gpu": J1,
               "parity_note": "J, V_1 and pol_t for every t of the K-partitioned run equal a 1-GPU context's bits"}
    dist.barrier()
    return res


def _kernel_profile(config):
    """ncu counts of the stage kernels for this workload (profiles/r02_stage_kernels.json), or None."""
    p = os.path.join(ROOT, "profiles", "r02_stage_kernels.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        d = json.load(f)
    return d.get(config)


def run_sweep(args):
    """cfg5: a batch of storage configurations (different pbar, eta -> different action grids) over one
    price model, solved by one batch context (esdp_create_batch); each instance = backward + 1024 simulated
    paths (1024 x 1024 = 1.05e6 paths over the whole sweep).  Rank r of N takes a stratified sample of the
    1024-configuration sweep (every (N n / 1024)-th configuration from offset r): with N n = 1024 the ranks
    cover the sweep exactly once.  Weak scaling, no data-path collective."""
    import numpy as np
    import torch
    import torch.distributed as dist
    import workloads
    import paper_2511_15629_b200 as E
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dev = torch.device("cuda", local)
    n = args.instances
    idx = workloads.cfg5_shard(rank, world, n)   # stratified over the sweep order
    insts = workloads.cfg5_instances(idx)
    batch = E.Batch(insts, force_brute=args.stencil == "brute",   # one graph: one expectation + one stencil launch per stage
                    ozaki=args.contract == "ozaki")
    stream = torch.cuda.Stream(device=dev)
    paths = 1024
    out_d = torch.empty(n * paths, dtype=torch.float64, device=dev)
    T, S, K = batch.T, batch.S, batch.K
    As = list(batch.A)
    cells = sum(T * S * K * a for a in As)
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
    J = batch.objective()
    launches = (batch.launch_count() + 1) * args.steps

    # end to end through the public API with host buffers: every step uploads the shared price model from
    # pinned host memory (esdp_batch_load_async: validation, H2D, sampling tables), solves, simulates and
    # reads every instance's J back to the host
    base = insts[0]
    lam_h = torch.from_numpy(np.ascontiguousarray(base.lam)).pin_memory()
    P_h = torch.from_numpy(np.ascontiguousarray(base.P)).pin_memory()
    pi_h = torch.from_numpy(np.ascontiguousarray(base.pi)).pin_memory()
    J_h = torch.zeros(n, dtype=torch.float64).pin_memory()
    h2d = (lam_h.numel() + P_h.numel() + pi_h.numel()) * 8

    def e2e_step(j):
        batch.load_async(lam_h.data_ptr(), P_h.data_ptr(), pi_h.data_ptr(), stream.cuda_stream)
        batch.backward_async(stream.cuda_stream)
        batch.simulate_dev(paths, 17 + j, out_d.data_ptr(), stream.cuda_stream)
        stream.synchronize()
        J_h.copy_(torch.from_numpy(batch.objective()))      # D2H of every instance's J

    for j in range(args.warmup):
        e2e_step(j)
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for j in range(args.steps):
        e2e_step(j)
    e2e_s = (time.perf_counter() - t0) / args.steps
    e2e_t = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(e2e_t, op=dist.ReduceOp.MAX)
    e2e_value = cells * world / float(e2e_t.item())

    # roofline of the dominant kernels (warm launches of stage T-1's batch kernels after the timed region)
    peaks, peak_kind = _peaks()
    hbm_peak = float(peaks["hbm_gbs"])
    kern = None
    if rank == 0:
        us_win = batch.kernel_time(1, 50)
        us_exp = batch.kernel_time(0, 50)
        outs = n * K * S
        win_bytes = 18.0 * outs
        exp_bytes = 8.0 * (2 * n * K * S + K * K)     # read V_{t+1}, write W_t, read P_t
        exp_flop = 2.0 * K * K * n * S
        kp = _kernel_profile("cfg5") if args.contract == "dmma" and args.stencil == "auto" and n == 128 else None
        kern = {"window": {"kernel": "window_batch_kernel", "us_per_launch": us_win, "bytes_per_launch": win_bytes,
                           "achieved": win_bytes / us_win / 1e3, "peak": hbm_peak, "unit": "GB/s",
                           "frac": win_bytes / us_win / 1e3 / hbm_peak, "traffic": None, "instr_per_output": None},
                "expectation": {"kernel": ("ozaki_contract_kernel (Ozaki u8 tcgen05, opt-in)" if batch.plan == 2 else
                                           "contract_dmma3_kernel") + " (one [K] x [n ld] GEMM per stage)",
                                "us_per_launch": us_exp, "bytes_per_launch": exp_bytes,
                                "hbm_frac": exp_bytes / us_exp / 1e3 / hbm_peak, "flop_per_launch": exp_flop,
                                "achieved_tflops": exp_flop / us_exp / 1e6,
                                "dmma_frac": exp_flop / us_exp / 1e6 / DMMA_PEAK_TFLOPS}}
        if kp and "window" in kp:   # ncu counts of this workload's launches (profiles/r02_stage_kernels.json)
            kern["window"]["traffic"] = kp["window"]["dram_bytes_per_launch"]
            kern["window"]["instr_per_output"] = kp["window"]["warp_inst_per_launch"] * 32.0 / outs
    batch.close()
    out = None
    if rank == 0:
        w = kern["window"]
        out = {"metric": "DP cell-updates/sec (T*S*K*A)", "value": cells * world / (ms * 1e-3), "unit": "cell-updates/s",
               "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
               "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
               "data": "synthetic (cfg2 price chain; cfg5 storage sweep)",
               "config": {"workload": "cfg5 sweep: %d storage configurations per GPU, a stratified sample of the "
                                      "1024-configuration sweep (pbar/delta in [10.42, 99], eta in [0.80, 0.99]; "
                                      "T=288, S=1001, K=100; A=%d..%d, mean %.1f), 1024 simulated paths each"
                                      % (n, min(As), max(As), float(np.mean(As))),
                          "instances_per_gpu": n, "sweep_indices": [idx[0], idx[-1], len(idx)],
                          "mean_A": float(np.mean(As)), "l2": "flushed between timed steps",
                          "sim_paths_per_step": n * paths * world,
                          "plan": "esdp_create_batch: per stage one [K] x [n ld] expectation (%s) + one window launch"
                                  % ("Ozaki u8 tcgen05, opt-in, tolerance 1e-9" if args.contract == "ozaki" else
                                     "FP64 DMMA, canonical chain")},
               "gpu_launches": launches, "J_mean": float(np.mean(J)),
               "roofline": {"bound": "hbm", "achieved": w["achieved"], "peak": hbm_peak, "unit": "GB/s",
                            "frac": w["frac"], "traffic": w["traffic"], "instr_per_output": w["instr_per_output"],
                            "kernel": w["kernel"],
                            "us_per_launch": w["us_per_launch"], "bytes_per_launch": w["bytes_per_launch"],
                            "work_per_launch": "18 B per output (m, k, s): read W_t, write V_t, pol_t",
                            "peak_note": "MEASURED_PEAKS.json hbm_gbs (%s)" % peak_kind},
               "roofline_kernels": kern,
               "e2e": {"value": e2e_value, "unit": "cell-updates/s", "h2d_bytes_per_step": h2d,
                       "d2h_bytes_per_step": 8 * n},
               "clocks": clk}
        if kp and "window" in kp:
            _issue_frac(out["roofline"], kp["window"]["warp_inst_per_launch"], clk, dev)
        if world == 1 and not args.no_cpu_baseline:
            out["cpu_baseline"] = cpu_baseline_sweep(insts, budget_s=args.cpu_budget)
    return out


def _issue_frac(roof, warp_inst, clk, dev):
    """Fraction of the SMs' warp-instruction issue slots (4 schedulers x SMs x SM clock) the kernel's
    instructions (ncu count per launch, profiles/) fill over its measured launch time: how close an
    issue-bound kernel is to its own instruction stream's bound."""
    import torch
    if roof is None or not warp_inst:
        return
    nsm = torch.cuda.get_device_properties(dev).multi_processor_count
    mhz = (clk or {}).get("sm_mhz") or (clk or {}).get("sm_max_mhz") or 1965.0
    slots = roof["us_per_launch"] * 1e-6 * nsm * 4 * mhz * 1e6
    roof["issue_frac"] = warp_inst / slots
    roof["issue_note"] = ("ncu warp instructions per launch / (launch time x %d SMs x 4 schedulers x %.0f MHz)"
                          % (nsm, mhz))


def cpu_baseline_sweep(insts, budget_s=15.0, n_inst=8):
    """The oracle on a bounded sample of the cfg5 step: n_inst configurations spread over the batch, the
    last few stages of each (every (k, i) row), extrapolated per cell (per-stage cost is constant)."""
    import oracle
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from helpers import to_oracle
    cores = os.cpu_count() or 1
    pick = [insts[(j * len(insts)) // n_inst] for j in range(min(n_inst, len(insts)))]
    prs = [to_oracle(x) for x in pick]
    t0 = time.perf_counter()
    oracle.backward(prs[0], t_stop=pick[0].T - 1, nthreads=cores)   # 2 stages to size the sample
    per_stage = max(time.perf_counter() - t0, 1e-3) / 2
    n_stages = int(max(2, min(pick[0].T, budget_s / (per_stage * len(pick)))))
    cells, t = 0, 0.0
    for x, pr in zip(pick, prs):
        S, A = oracle.dims(pr)
        t0 = time.perf_counter()
        oracle.backward(pr, t_stop=x.T - n_stages + 1, nthreads=cores)
        t += time.perf_counter() - t0
        cells += n_stages * S * x.K * A
    return {"value": cells / t, "unit": "cell-updates/s", "cores": cores, "kind": "oracle",
            "sample": f"oracle backward of {len(pick)} configurations spread over the batch, the last {n_stages} "
                      f"of {pick[0].T} stages each (all K*S rows, OpenMP {cores} threads), {t:.2f} s"}


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
            "config": {"workload": _workload_name(args), "sample": sample},
            "cpu_baseline": {"value": value, "unit": "cell-updates/s", "cores": cores, "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": value, "unit": "cell-updates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def _self_launch(n):
    """--gpus N > 1 without a torchrun environment: run this script under torch.distributed.run, one process
    per GPU on this node (rendezvous on 127.0.0.1), and exit with its status."""
    import socket
    import torch
    if torch.cuda.device_count() < n:
        print(f"bench.py: --gpus {n} but only {torch.cuda.device_count()} CUDA devices are visible", file=sys.stderr)
        return 2
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="cfg2", choices=sorted(WORKLOAD) + ["cfg5"])
    ap.add_argument("--instances", type=int, default=128,
                    help="cfg5: storage configurations per GPU (a stratified sample of the 1024-configuration sweep; "
                         "8 GPUs x 128 = the whole sweep)")
    ap.add_argument("--t3-hours", type=float, default=100.0, help="table3: battery duration (hours)")
    ap.add_argument("--t3-delta", type=float, default=0.01, help="table3: SoC step (MWh)")
    ap.add_argument("--paths", type=int, default=65536)
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--ref-stages", type=int, default=24)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--kernel-events", type=int, default=1,
                    help="per-phase split of the backward from a separate context with CUDA events around ~16 stages")
    ap.add_argument("--bids", choices=["fused", "after", "with-sim"], default="fused",
                    help="bid curves as side branches of the backward graph (fused), one kernel after it, or one "
                         "kernel on a side stream concurrent with the simulation")
    ap.add_argument("--contract", choices=["dmma", "ozaki"], default="dmma",
                    help="cfg5: expectation plan (ozaki: ESDP_CONTRACT_OZAKI, the NEXT-4 tcgen05 path, not bit-exact)")
    ap.add_argument("--stencil", choices=["auto", "brute"], default="auto",
                    help="auto: exact sliding-window stencil where it applies; brute: every (i, a) cell")
    ap.add_argument("--mode", choices=["instances", "kpart"], default=None,
                    help="N>1: one K-partitioned instance (kpart, the default main line, strong scaling) or "
                         "independent instances per rank (instances, weak)")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(_self_launch(args.gpus))
    if args.warmup < 3 and args.impl == "ours":
        print("warning: --warmup < 3 violates the timing rules", file=sys.stderr)
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.impl == "reference":
        out = run_reference(args)   # rank 0 only; the other ranks exit without work
    else:
        import torch
        import torch.distributed as dist
        local = int(os.environ.get("LOCAL_RANK", "0"))
        torch.cuda.set_device(local)
        if world > 1:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        if args.config == "cfg5":
            out = run_sweep(args)
        else:
            mode = args.mode or ("kpart" if world > 1 else "instances")
            out = run_ours(args, mode)
            if world > 1 and args.mode is None:   # the instance-sharded (weak) number beside the main line
                extra_args = argparse.Namespace(**vars(args))
                extra_args.kernel_events = 0
                extra = run_ours(extra_args, "instances")
                if rank == 0:
                    out["instances_weak"] = {k: extra[k] for k in ("value", "unit", "ms_per_step", "scaling", "e2e")}
                    out["instances_weak"]["parallelism"] = extra["config"]["parallelism"]
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
    if out is not None:
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
