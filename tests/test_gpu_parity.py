"""GPU parity: the CUDA path (through the C ABI) against the FP64 oracle on the same seeded inputs.

Bar: V, W, J bit-identical (the kernels use the oracle's exact association and the
canonical fma chain, so any difference is a bug; the north_star tolerance 1e-9 relative is asserted
as well), policy and bid-curve vertex indices bit-exact, bid prices bit-exact, per-path simulation
profits bit-exact."""
import math

import numpy as np
import pytest

import oracle
import workloads
from helpers import to_oracle

pytestmark = pytest.mark.gpu

import paper_2511_15629_b200 as E  # no skip: a missing library must fail loudly


def _gpu(inst, brute=False, dmma=True, keep=True):
    return E.Solver(inst, keep_values=keep, force_brute=brute, dmma=dmma)


def _compare_all(inst, nthreads=8, stages=None, brute=False, expect_window=None, dmma=True):
    pr = to_oracle(inst)
    ref = oracle.backward(pr, nthreads=nthreads)
    with _gpu(inst, brute, dmma) as s:
        if expect_window is not None:
            assert (s.stencil_kind & 1) == int(expect_window)
        if brute:
            assert (s.stencil_kind & 1) == 0
        J = s.backward()
        assert np.array_equal(s.actions(), oracle.actions(pr))
        ts = range(1, inst.T + 1) if stages is None else stages
        for t in ts:
            V, W = s.values(t)
            pol = s.policy(t)
            assert np.array_equal(W, ref.W[t - 1]), f"W_{t} differs: max |d| {np.max(np.abs(W - ref.W[t-1]))}"
            assert np.array_equal(V, ref.V[t - 1]), f"V_{t} differs: max |d| {np.max(np.abs(V - ref.V[t-1]))}"
            assert np.array_equal(pol, ref.pol[t - 1]), f"pol_{t} differs at {np.argwhere(pol != ref.pol[t-1])[:5]}"
        assert J == ref.J
        assert abs(J - ref.J) <= 1e-9 * max(1.0, abs(ref.J))
    return ref


@pytest.mark.parametrize("brute", [False, True])
@pytest.mark.parametrize("seed", range(40))
def test_random_small_instances(seed, brute):
    kind = [workloads.PAYOFF_LINEAR, workloads.PAYOFF_LINEAR_MINUS_G, workloads.PAYOFF_TABLE][seed % 3]
    inst = workloads.random_instance(seed, S_max=40 if seed % 2 else 600, T=4 + seed % 3, K=1 + seed % 4)
    S, A = oracle.dims(to_oracle(inst))
    inst.payoff_kind = kind
    if kind == workloads.PAYOFF_LINEAR_MINUS_G:
        inst.g = workloads.random_g(seed, A, 20.0)
    elif kind == workloads.PAYOFF_TABLE:
        inst.g = workloads.random_table(seed, inst.T, inst.K, A)
    _compare_all(inst, brute=brute)


@pytest.mark.parametrize("dmma", [True, False])
@pytest.mark.parametrize("K", [8, 13, 30, 37, 64])
def test_expectation_tensor_cores_bitexact(K, dmma):
    """FP64 DMMA (mma.sync m8n8k4) expectation: K not a multiple of 4, rows not a multiple of 8, ragged
    columns; bit-identical to the oracle's sequential fma chain (and the DFMA kernel likewise)."""
    inst = workloads.random_instance(1000 + K, T=4, K=K, S_max=300, rank1=False)
    _compare_all(inst, dmma=dmma)


@pytest.mark.parametrize("brute", [False, True])
@pytest.mark.parametrize("name", ["cfg1a", "cfg1b", "cfg1b-rank1", "cfg1a-rank1"])
def test_cfg1(name, brute):
    _compare_all(workloads.cfg1(name[4], rank1=name.endswith("rank1")), brute=brute,
                 expect_window=None if brute else True)


@pytest.mark.parametrize("brute", [False, True])
@pytest.mark.parametrize("S_over", [2, 50, 150, 255, 256, 257, 511, 777, 1001, 2001])
def test_tiles_and_ragged_tails(S_over, brute):
    """Several 256-column tiles plus a ragged tail; cfg2-like offsets (also S smaller than the
    action span, where most actions are infeasible)."""
    inst = workloads.cfg2(T=6, K=7)
    inst.sbar = float(S_over - 1)
    inst.s0 = 0.0
    _compare_all(inst, brute=brute)


@pytest.mark.parametrize("brute", [False, True])
def test_edge_cases(brute):
    # T = 1, K = 1, minimal grid (S = 2)
    inst = workloads.random_instance(5, T=1, K=1, S_max=3)
    inst.sbar, inst.delta, inst.s0 = 1.0, 1.0, 0.0
    _compare_all(inst, brute=brute)
    # pbar far larger than sbar: most actions infeasible everywhere (dead actions)
    inst = workloads.random_instance(6, T=3, K=2, S_max=5)
    inst.pbar = 50.0 * inst.sbar
    _compare_all(inst, brute=brute)
    # user action grid: every action off the lattice (all interpolated), off-grid s0
    inst = workloads.random_instance(7, T=5, K=3, S_max=30)
    inst.actions = np.array([-0.93, -0.41, -0.07, 0.0, 0.13, 0.52, 0.99]) * inst.pbar
    inst.s0 = inst.sbar * 0.37
    _compare_all(inst, brute=brute)
    # zero prices: every candidate ties, the smallest feasible action must be chosen
    inst = workloads.cfg1("b")
    inst.lam = np.zeros_like(inst.lam)
    _compare_all(inst, brute=brute)
    # integer prices on an eta = 1 lattice: many exact ties
    inst = workloads.cfg1("a")
    inst.lam = np.round(inst.lam / 10.0)
    _compare_all(inst, brute=brute)


def test_cfg2_full_size():
    """BASELINE configs[1] at full size (T=288, S=1001, A=201, K=100), in the launch configuration
    bench.py times (sliding-window stencil): every V_t, W_t, pol_t compared element by element."""
    _compare_all(workloads.cfg2(), nthreads=16, expect_window=True)


def test_cfg2_full_size_bruteforce():
    _compare_all(workloads.cfg2(), nthreads=16, brute=True)


@pytest.mark.parametrize("name", ["cfg1b", "cfg1b-rank1", "cfg2-small"])
def test_dist_path_single_rank_bitexact(name):
    """esdp_create_dist with world = 1: the K-partitioned graph with the per-stage NCCL all-gather of V_t
    and pol_t (a copy on one rank) gives the oracle's results bit for bit."""
    inst = workloads.cfg2(T=24, K=20) if name == "cfg2-small" else workloads.cfg1("b", rank1=name.endswith("rank1"))
    pr = to_oracle(inst)
    ref = oracle.backward(pr, nthreads=8)
    nid = E.esdp_nccl_unique_id()
    with E.Solver(inst, keep_values=True, dist=(1, 0, nid)) as s:
        assert s.stencil_kind & 2                # DMMA expectation (the probe passed)
        assert s.backward() == ref.J
        for t in range(1, inst.T + 1):
            V, W = s.values(t)
            assert np.array_equal(V, ref.V[t - 1]) and np.array_equal(W, ref.W[t - 1])
            assert np.array_equal(s.policy(t), ref.pol[t - 1])
        per, m, v = s.simulate(500, 3)
        per_ref, _, _ = oracle.simulate(pr, ref.pol, 500, 3)
        assert np.array_equal(per, per_ref)


def test_cfg2_full_size_dfma_expectation():
    _compare_all(workloads.cfg2(), nthreads=16, dmma=False)


def test_cfg2_no_keep_values():
    """Without ESDP_KEEP_VALUES the backward ping-pongs V/W; V_1, every policy and J are unchanged."""
    inst = workloads.cfg2(T=40, K=30)
    pr = to_oracle(inst)
    ref = oracle.backward(pr, nthreads=8)
    with _gpu(inst, keep=False) as s:
        assert s.backward() == ref.J
        V1 = E.esdp_values(s.ctx, 1, want_W=False)
        assert np.array_equal(V1, ref.V[0])
        for t in range(1, inst.T + 1):
            assert np.array_equal(s.policy(t), ref.pol[t - 1])


@pytest.mark.parametrize("rank1", [False, True])
def test_graph_without_pdl(rank1):
    """The graph plan without programmatic dependent launch (ESDP_NO_PDL) gives the same bits as the
    default late-trigger PDL chain."""
    inst = workloads.cfg2(T=30, K=30, rank1=rank1)
    pr = to_oracle(inst)
    ref = oracle.backward(pr, nthreads=16)
    with E.Solver(inst, pdl=False) as s:
        assert s.backward() == ref.J
        for t in range(1, inst.T + 1):
            V, W = s.values(t)
            assert np.array_equal(V, ref.V[t - 1]) and np.array_equal(W, ref.W[t - 1])
            assert np.array_equal(s.policy(t), ref.pol[t - 1])


@pytest.mark.parametrize("rank1", [False, True])
def test_async_load_overlaps_and_matches(rank1):
    """esdp_load_async: new prices and transitions uploaded in stage chunks while the backward runs (the
    graph waits per chunk) give the oracle's bits for the new data; repeated async loads alternate
    between two instances; the simulation's sampling tables follow the new P."""
    a = workloads.cfg2(T=40, K=20, rank1=rank1)
    b = workloads.cfg2(T=40, K=20, rank1=rank1)
    lam_b, _, _ = workloads.price_chain(a.T, a.K, 5.0 / 60.0, seed=workloads.SEED_BASE + 4242)
    b.lam = lam_b
    if not rank1:
        rng = np.random.default_rng(7)
        Pb = a.P * rng.uniform(0.5, 1.5, a.P.shape)
        b.P = Pb / Pb.sum(axis=2, keepdims=True)
    refs = [oracle.backward(to_oracle(x), nthreads=16) for x in (a, b)]
    sims = {}
    with E.Solver(a) as s:
        for rep in range(4):
            x, ref = ((a, refs[0]), (b, refs[1]))[rep % 2]
            keep = E.esdp_load_async(s.ctx, lam=x.lam, P=x.P, pi=x.pi)
            J = s.backward()
            del keep
            assert J == ref.J
            for t in (1, x.T // 2, x.T):
                V, W = s.values(t)
                assert np.array_equal(V, ref.V[t - 1]) and np.array_equal(W, ref.W[t - 1])
                assert np.array_equal(s.policy(t), ref.pol[t - 1])
            m = s.simulate(4096, seed=5, per_path=False)[1]
            key = rep % 2
            if key in sims:
                assert m == sims[key]
            sims[key] = m
        assert sims[0] != sims[1]


def test_cfg2_rank1_full_size():
    _compare_all(workloads.cfg2(rank1=True), nthreads=16, expect_window=True)


def test_table3_largest_row_shape():
    """The paper's Table 3 largest row (bench.py --config table3) at its full per-stage shape: S = 10001,
    A = 203, R = K = 200 rank-1 price samples, on a 48-hour horizon (the stage's launch configuration -- grid,
    four outputs per thread, the rank-1 GEMV on the DMMA path -- does not depend on T): every stage's W, V and
    policy bit-identical to the oracle's."""
    inst = workloads.table3(T=48)
    assert inst.K == 200 and inst.P is None
    ref = _compare_all(inst, nthreads=16, expect_window=True)
    assert ref.V[0].shape == (200, 10001)


def test_table3_largest_row_full_year():
    """The same row over the whole year (T = 8784) as bench.py times it (no ESDP_KEEP_VALUES; the oracle's
    full solve would take ~15 CPU-minutes, so the per-stage bits are the shape test's above): J equals the
    oracle's objective (Eq. 6 at t = 0) of the GPU's V_1, V_1 is finite on the whole grid (the zero action is
    always feasible, Alg. 1 line 8), and every policy entry of stage 1 is an action index."""
    inst = workloads.table3()
    pr = to_oracle(inst)
    with _gpu(inst, keep=False) as s:
        J = s.backward()
        V1 = E.esdp_values(s.ctx, 1, want_W=False)
        assert V1.shape == (200, 10001) and np.all(np.isfinite(V1))
        assert J == oracle.objective(pr, V1)
        pol1 = s.policy(1)
        assert pol1.shape == (200, 10001) and pol1.min() >= 0 and pol1.max() < len(oracle.actions(pr))


@pytest.mark.parametrize("delta", [0.1, 0.01])
def test_table1_deterministic_year(delta):
    """NEXT-3 (Table 1 analog): K = 1, T = 8784 hourly stages, the paper's 4-h battery at
    delta = 0.10 (S=41, A=22) and 0.01 (S=401, A=203); every stage bit-identical to the oracle."""
    inst = workloads.table1_deterministic(delta)
    _compare_all(inst, nthreads=16)


def test_cfg4_slice():
    """BASELINE configs[3] per-stage shape (S=2001, A=401, K=200, a distinct P_t per stage) on a
    6-stage horizon, compared in full."""
    inst = workloads.cfg4(T=6)
    _compare_all(inst, nthreads=16, expect_window=True)


@pytest.mark.parametrize("brute", [False, True])
def test_cfg3i_table2_analog(brute):
    """cfg3i, the Table-2 analog: K = 1, T = 72 hourly, every price level-shifted <= 0,
    s0 = sbar, eta = sqrt(0.85) (interpolated endpoints).  Every V_t, W_t, pol_t and J bit-identical to the
    oracle (whose LP / MILP ordering pins are in test_oracle_backward.py), on both stencils; with prices
    <= 0 charging is paid or free, so J >= 0 and the last stage never discharges at a negative price."""
    inst = workloads.cfg3_small()
    assert inst.lam.max() <= 0.0
    ref = _compare_all(inst, brute=brute, expect_window=not brute)
    assert ref.J >= 0.0
    acts = oracle.actions(to_oracle(inst))
    lam_T = inst.lam[-1, 0]
    if lam_T < 0:
        assert np.all(acts[ref.pol[-1][0]] <= 0.0)


def test_cfg3_nonconcave_payoff_and_bids():
    """configs[2]: negative prices, degradation + fixed cycling cost (non-concave payoff), monotone
    bid curves (bit-exact vertices and prices) on a sample of (t, i, k)."""
    base = workloads.cfg2(T=2, K=2)
    act = oracle.actions(to_oracle(base))
    inst = workloads.cfg3_gpu(act, T=48, K=40)
    ref = _compare_all(inst)
    pr = to_oracle(inst)
    rng = np.random.default_rng(3)
    req = np.stack([rng.integers(1, inst.T + 1, 400), rng.integers(0, inst.S, 400), rng.integers(0, inst.K, 400)], 1)
    req[:10, 1] = [0, 1, 2, 998, 999, 1000, 500, 94, 95, 105]
    with _gpu(inst) as s:
        s.backward()
        out = s.bidcurves(req)
    for j, (t, i, k) in enumerate(req):
        c = oracle.bidcurve(pr, ref.W, int(t), int(i), int(k))
        n = out["nvert"][j]
        assert n == c["nvert"]
        assert np.array_equal(out["vert"][j, :n], c["vert"])
        assert np.array_equal(out["q"][j, :n], c["q"])
        assert np.array_equal(out["price"][j, :n - 1], c["price"])
        assert np.all(np.diff(out["price"][j, :n - 1]) >= 0)


@pytest.mark.parametrize("rank1", [False, True])
def test_cfg3_window_affine_degradation(rank1):
    """NEXT-1 for lambda p - g(p) with g affine on each side (cfg3: 2|p| + 25 [p != 0]): the exact
    sliding-window stencil applies (slopes beta +- g1, constants g0) and stays bit-identical to the
    oracle's brute force at full cfg3ii size; forcing brute force gives the same bits."""
    base = workloads.cfg2(T=2, K=2)
    inst = workloads.cfg3_gpu(oracle.actions(to_oracle(base)), T=24, K=100, rank1=rank1)
    _compare_all(inst, nthreads=16, expect_window=True)
    _compare_all(inst, nthreads=16, brute=True)


@pytest.mark.parametrize("which", ["cfg2", "cfg3"])
def test_window_unimodal_and_level_tables(which):
    """The window stencil answers a unimodal run table from its peak and builds sparse-table levels only
    for the others; both give the oracle's bits.  Linear payoff (cfg2 shape): every
    table unimodal.  cfg3's fixed cycling cost makes W non-concave: many tables take the level path."""
    base = workloads.cfg2(T=6, K=24)
    inst = base if which == "cfg2" else workloads.cfg3_gpu(oracle.actions(to_oracle(base)), T=6, K=24)
    with _gpu(inst) as s:
        E.esdp_window_level_tables(s.ctx)        # reset
    _compare_all(inst, nthreads=16, expect_window=True)
    with _gpu(inst) as s:
        E.esdp_window_level_tables(s.ctx)
        s.backward()
        lvl = E.esdp_window_level_tables(s.ctx)
        tables = inst.T * inst.K * ((s.S + 255) // 256) * 2
    if which == "cfg2":
        assert lvl == 0, (lvl, tables)
    else:
        assert 0.1 * tables < lvl < tables, (lvl, tables)


@pytest.mark.parametrize("seed", range(12))
def test_window_affine_g_random(seed):
    """Random instances with g = per-side affine (random slopes and fixed costs, g(0) = 0) use the window
    plan and match the oracle bit for bit; a non-affine g loaded later (esdp_load) only widens the
    exactness margin (canonical fallbacks), never changes a bit."""
    rng = np.random.default_rng(900 + seed)
    inst = workloads.random_instance(900 + seed, T=4, K=1 + seed % 5, S_max=700, rank1=bool(seed % 2))
    pr0 = to_oracle(inst)
    act = oracle.actions(pr0)
    cc, cd = rng.uniform(-3, 3, 2)
    fc, fd = rng.uniform(0, 30, 2)
    g = np.where(act < 0, -cc * act + fc, np.where(act > 0, cd * act + fd, 0.0))
    inst.payoff_kind = workloads.PAYOFF_LINEAR_MINUS_G
    inst.g = g
    S, A = oracle.dims(pr0)
    _compare_all(inst, expect_window=None)
    with _gpu(inst) as s:
        if not s.stencil_kind & 1:   # too few actions on a side for the window plan
            return
        g2 = g + workloads.random_g(seed, A, 1.0)
        E.esdp_load(s.ctx, g=g2)
        inst2 = workloads.Instance(**{**inst.__dict__, "g": g2})
        ref2 = oracle.backward(to_oracle(inst2))
        assert s.backward() == ref2.J
        for t in range(1, inst.T + 1):
            V, _ = s.values(t)
            assert np.array_equal(V, ref2.V[t - 1]) and np.array_equal(s.policy(t), ref2.pol[t - 1])


@pytest.mark.parametrize("name", ["cfg1b", "cfg1b-rank1", "cfg3"])
def test_fused_bidcurves_in_backward(name):
    """esdp_set_bid_requests: curves extracted inside the backward graph (side branch per stage, unsorted
    requests over all stages) equal the oracle's bit for bit, on every backward pass."""
    import torch
    if name == "cfg3":
        base = workloads.cfg2(T=2, K=2)
        inst = workloads.cfg3_gpu(oracle.actions(to_oracle(base)), T=30, K=20)
    else:
        inst = workloads.cfg1("b", rank1=name.endswith("rank1"))
    pr = to_oracle(inst)
    ref = oracle.backward(pr)
    rng = np.random.default_rng(5)
    n = 3000
    req = np.stack([rng.integers(1, inst.T + 1, n), rng.integers(0, inst.S, n), rng.integers(0, inst.K, n)], 1)
    with _gpu(inst) as s:
        cap = s.A
        nv = torch.zeros(n, dtype=torch.int32, device="cuda")
        vert = torch.zeros(cap * n, dtype=torch.int16, device="cuda")
        q = torch.zeros(cap * n, dtype=torch.float64, device="cuda")
        price = torch.zeros(cap * n, dtype=torch.float64, device="cuda")
        E.esdp_set_bid_requests(s.ctx, req, cap, nv.data_ptr(), vert.data_ptr(), q.data_ptr(), price.data_ptr())
        for rep in range(2):
            nv.zero_(); vert.zero_(); price.zero_()
            s.backward()
            torch.cuda.synchronize()
            nvh = nv.cpu().numpy(); vh = vert.cpu().numpy().reshape(cap, n); ph = price.cpu().numpy().reshape(cap, n)
            qh = q.cpu().numpy().reshape(cap, n)
            for j in range(0, n, 7):
                t, i, k = (int(x) for x in req[j])
                c = oracle.bidcurve(pr, ref.W, t, i, k)
                m = nvh[j]
                assert m == c["nvert"]
                assert np.array_equal(vh[:m, j], c["vert"]) and np.array_equal(qh[:m, j], c["q"])
                assert np.array_equal(ph[:m - 1, j], c["price"])
        E.esdp_set_bid_requests(s.ctx, np.zeros((0, 3), np.int32), cap, None, None, None, None)
        assert s.backward() == ref.J
        # requests on a few stages only (some side streams unused)
        few = req[np.isin(req[:, 0], [1, inst.T])]
        E.esdp_set_bid_requests(s.ctx, few, cap, nv.data_ptr(), vert.data_ptr(), q.data_ptr(), price.data_ptr())
        assert s.backward() == ref.J


@pytest.mark.parametrize("name", ["cfg1b", "cfg1b-rank1"])
def test_bidcurves_cfg1(name):
    inst = workloads.cfg1("b", rank1=name.endswith("rank1"))
    pr = to_oracle(inst)
    ref = oracle.backward(pr)
    req = np.array([(t, i, k) for t in range(1, inst.T + 1) for i in range(0, inst.S, 7) for k in range(inst.K)])
    with _gpu(inst) as s:
        s.backward()
        out = s.bidcurves(req)
    for j, (t, i, k) in enumerate(req):
        c = oracle.bidcurve(pr, ref.W, int(t), int(i), int(k))
        n = out["nvert"][j]
        assert n == c["nvert"] and np.array_equal(out["vert"][j, :n], c["vert"])
        assert np.array_equal(out["price"][j, :n - 1], c["price"])


@pytest.mark.parametrize("fused", [False, True])
def test_bidcurves_wide_grid_global_stack(fused):
    """A > 255 (cfg4's grid, A = 401: the hull stack lives in the vertex row in global memory): vertices,
    quantities and prices bit-identical to the oracle, on demand and fused into the backward graph, every
    stage of a short horizon and SoC rows across the grid (ragged S = 2001)."""
    inst = workloads.cfg4(T=3, K=4)
    pr = to_oracle(inst)
    ref = oracle.backward(pr, nthreads=16)
    req = np.array([(t, i, k) for t in range(1, inst.T + 1) for i in list(range(0, 2001, 37)) + [1999, 2000]
                    for k in (0, 3)], dtype=np.int32)
    with _gpu(inst) as s:
        assert s.A == 401
        if fused:
            import torch
            n, cap = len(req), s.A
            nv = torch.zeros(n, dtype=torch.int32, device="cuda")
            vt = torch.zeros(cap * n, dtype=torch.int16, device="cuda")
            qq = torch.zeros(cap * n, dtype=torch.float64, device="cuda")
            pp = torch.zeros(cap * n, dtype=torch.float64, device="cuda")
            E.esdp_set_bid_requests(s.ctx, req, cap, nv.data_ptr(), vt.data_ptr(), qq.data_ptr(), pp.data_ptr())
            s.backward()
            torch.cuda.synchronize()
            nvh = nv.cpu().numpy()
            vth = vt.cpu().numpy().reshape(cap, n).T
            pph = pp.cpu().numpy().reshape(cap, n).T
            qqh = qq.cpu().numpy().reshape(cap, n).T
        else:
            s.backward()
            out = s.bidcurves(req)
            nvh, vth, pph, qqh = out["nvert"], out["vert"], out["price"], out["q"]
    acts = oracle.actions(pr)
    for j, (t, i, k) in enumerate(req):
        c = oracle.bidcurve(pr, ref.W, int(t), int(i), int(k))
        nn = int(nvh[j])
        assert nn == c["nvert"], (t, i, k)
        assert np.array_equal(vth[j, :nn], c["vert"]), (t, i, k)
        assert np.array_equal(pph[j, :nn - 1], c["price"]), (t, i, k)
        assert np.array_equal(qqh[j, :nn], acts[c["vert"]]), (t, i, k)


@pytest.mark.parametrize("name", ["cfg1b", "cfg1b-rank1", "cfg2"])
def test_simulation_per_path_bitexact(name):
    inst = workloads.cfg2(T=48, K=30) if name == "cfg2" else workloads.cfg1("b", rank1=name.endswith("rank1"))
    pr = to_oracle(inst)
    ref = oracle.backward(pr, nthreads=8)
    n = 3000
    per_ref, m_ref, v_ref = oracle.simulate(pr, ref.pol, n, seed=777)
    with _gpu(inst) as s:
        J = s.backward()
        per, m, v = s.simulate(n, 777)
    assert np.array_equal(per, per_ref)
    assert abs(m - m_ref) <= 1e-12 * max(1.0, abs(m_ref))
    assert abs(v - v_ref) <= 1e-9 * max(1.0, abs(v_ref))
    assert abs(m - J) <= 5 * math.sqrt(v / n) + 1e-9


@pytest.mark.parametrize("K", [40, 5])
def test_simulation_sampler_edge_tables(K):
    """The one-load sampler (DESIGN.md §5 a7) against the definition on transition rows built to hit every
    guide case: exact zeros (empty states the one-boundary step skips), clusters of 1e-12..1e-15
    probabilities (several boundaries in one bucket: the scan), dominant entries (pure buckets), three
    distinct slices repeated over the stages (table dedupe) and a pi_1 with zeros; per-path profits
    bit-identical to the oracle."""
    rng = np.random.default_rng(11 + K)
    base = workloads.cfg2(T=12, K=K)

    def row():
        w = np.zeros(K)
        sup = rng.choice(K, size=max(2, K // 2), replace=False)
        w[sup] = rng.choice([1.0, 0.3, 1e-12, 3e-13, 1e-15], size=len(sup))
        w[sup[0]] = 1.0
        return w / w.sum()

    slices = [np.stack([row() for _ in range(K)]) for _ in range(3)]
    base.P = np.ascontiguousarray(np.stack([slices[t % 3] for t in range(base.T - 1)]))
    pi = row()
    base.pi = pi
    pr = to_oracle(base)
    ref = oracle.backward(pr, nthreads=8)
    n = 4000
    per_ref, _, _ = oracle.simulate(pr, ref.pol, n, seed=4242)
    with _gpu(base) as s:
        assert s.backward() == ref.J
        per, _, _ = s.simulate(n, 4242)
    assert np.array_equal(per, per_ref)


def test_load_new_prices_and_repeat():
    """esdp_load replaces the stochastic inputs in place; repeated solves are bit-identical."""
    a = workloads.cfg1("b")
    b = workloads.cfg1("b")
    b.lam = b.lam * 1.3 + 2.0
    ref_b = oracle.backward(to_oracle(b))
    with _gpu(a) as s:
        J1 = s.backward()
        E.esdp_load(s.ctx, lam=b.lam)
        Jb = s.backward()
        Jb2 = s.backward()
        assert Jb == ref_b.J and Jb2 == Jb
        V, W = s.values(1)
        assert np.array_equal(V, ref_b.V[0])
        with pytest.raises(E.EsdpError) as ei:
            bad = b.lam.copy(); bad[0, 0] = np.nan
            E.esdp_load(s.ctx, lam=bad)
        assert ei.value.status == E.ESDP_E_DATA


def test_state_errors():
    inst = workloads.cfg1("b")
    with _gpu(inst) as s:
        with pytest.raises(E.EsdpError) as ei:
            s.values(1)
        assert ei.value.status == E.ESDP_E_STATE
        s.backward()
        with pytest.raises(E.EsdpError):
            s.values(inst.T + 1)
        with pytest.raises(E.EsdpError):
            s.bidcurves(np.array([[1, 10_000, 0]]))


@pytest.mark.parametrize("mode", ["physical", "clear"])
@pytest.mark.parametrize("name", ["cfg1a", "cfg1b", "cfg1b-rank1", "cfg3", "random-g"])
def test_simulation_modes_bitexact(name, mode):
    """a7's other modes on the GPU equal the oracle path by path: physical re-optimisation at the real
    SoC (off-grid interpolation of W_t) and bid-curve clearing at the realised price."""
    if name == "cfg3":
        base = workloads.cfg2(T=2, K=2)
        inst = workloads.cfg3_gpu(oracle.actions(to_oracle(base)), T=20, K=12)
    elif name == "random-g":
        inst = workloads.random_instance(61, T=6, K=3, S_max=200)
        act = oracle.actions(to_oracle(inst))
        inst.payoff_kind = workloads.PAYOFF_LINEAR_MINUS_G
        inst.g = workloads.random_g(61, len(act), 3.0)
        inst.s0 = inst.sbar * 0.37
    else:
        inst = workloads.cfg1(name[4], rank1=name.endswith("rank1"))
        inst.s0 = inst.sbar * 0.5 + 0.3 * inst.delta          # off-grid start (physical mode's real SoC)
    pr = to_oracle(inst)
    ref = oracle.backward(pr)
    m = oracle.SIM_PHYSICAL if mode == "physical" else oracle.SIM_CLEAR_BIDS
    n = 2500
    want, wm, wv = oracle.simulate_mode(pr, ref.pol, ref.W, m, n, seed=31)
    with _gpu(inst) as s:
        s.backward()
        got, gm, gv = s.simulate(n, 31, mode=E.ESDP_SIM_PHYSICAL if mode == "physical" else E.ESDP_SIM_CLEAR_BIDS)
    assert np.array_equal(got, want)
    assert gm == pytest.approx(wm, rel=1e-12)


def test_simulation_modes_state_errors():
    inst = workloads.cfg1("b")
    with E.Solver(inst, keep_values=False) as s:
        s.backward()
        with pytest.raises(E.EsdpError) as e:
            s.simulate(10, 1, mode=E.ESDP_SIM_PHYSICAL)
        assert e.value.status == E.ESDP_E_STATE


@pytest.mark.parametrize("rank1", [False, True])
def test_pipelined_double_buffered_loads(rank1):
    """Pipelined steps: load(j+1) is issued while solve j runs and before solve j's results are read;
    the results of solve j (J, values, policy, simulation) stay those of inputs j, and every solve
    matches the oracle on its own inputs.  NULL arrays keep the newest inputs."""
    import torch
    insts = []
    for j in range(4):
        x = workloads.cfg2(T=24, K=12, rank1=rank1)
        x.lam, _, _ = workloads.price_chain(x.T, x.K, 5.0 / 60.0, seed=workloads.SEED_BASE + 900 + j)
        insts.append(x)
    refs = [oracle.backward(to_oracle(x), nthreads=16) for x in insts]
    sims = [oracle.simulate(to_oracle(x), r.pol, 512, seed=4)[0] for x, r in zip(insts, refs)]
    with E.Solver(insts[0]) as s:
        keep = [E.esdp_load_async(s.ctx, lam=insts[0].lam)]
        for j in range(4):
            E.esdp_backward_async(s.ctx)
            if j + 1 < 4:
                keep.append(E.esdp_load_async(s.ctx, lam=insts[j + 1].lam))   # overlaps solve j
            torch.cuda.synchronize()
            assert E.esdp_objective(s.ctx) == refs[j].J
            V, W = s.values(1)
            assert np.array_equal(V, refs[j].V[0]) and np.array_equal(W, refs[j].W[0])
            assert np.array_equal(s.policy(insts[j].T // 2), refs[j].pol[insts[j].T // 2 - 1])
            per, _, _ = s.simulate(512, seed=4)
            assert np.array_equal(per, sims[j])
        # two loads without a solve: the second replaces the first; NULL keeps the newest inputs
        E.esdp_load(s.ctx, lam=insts[1].lam)
        E.esdp_load(s.ctx, lam=insts[2].lam)
        assert s.backward() == refs[2].J
        E.esdp_load(s.ctx, pi=insts[2].pi)
        assert s.backward() == refs[2].J


def test_cfg3_full_size_every_stage():
    """cfg3ii at full size (T=288, S=1001, A=201, K=100; non-concave payoff on the window plan): every
    stage bit-identical to the oracle."""
    base = workloads.cfg2(T=2, K=2)
    inst = workloads.cfg3_gpu(oracle.actions(to_oracle(base)))
    _compare_all(inst, nthreads=16, expect_window=True)


def test_cfg4_full_year_sampled_stages():
    """cfg4 at full size (T=8760, S=2001, A=401, K=200; a distinct P_t per stage) in the bench's launch
    configuration: every sampled stage t equals the oracle's stage computed from the GPU's own V_{t+1}
    (each stage is a pure function of V_{t+1}), the last stages from scratch, and J from V_1."""
    inst = workloads.cfg4()
    pr = to_oracle(inst)
    T = inst.T
    WT, VT, polT = oracle.stage(pr, T, 0, inst.K, None, nthreads=16)          # from scratch
    WT1, VT1, polT1 = oracle.stage(pr, T - 1, 0, inst.K, VT, nthreads=16)
    with _gpu(inst) as s:
        J = s.backward()
        for t, (Wr, Vr, pr_) in ((T, (WT, VT, polT)), (T - 1, (WT1, VT1, polT1))):
            V, W = s.values(t)
            assert np.array_equal(W, Wr) and np.array_equal(V, Vr)
            assert np.array_equal(s.policy(t), pr_)
        for t in (T - 2, 4380, 1234, 2, 1):
            Vn, _ = s.values(t + 1)
            W_ref, V_ref, pol_ref = oracle.stage(pr, t, 0, inst.K, Vn, nthreads=16)
            V, W = s.values(t)
            assert np.array_equal(W, W_ref), t
            assert np.array_equal(V, V_ref), t
            assert np.array_equal(s.policy(t), pol_ref), t
        V1, _ = s.values(1)
        assert J == oracle.objective(pr, V1)


@pytest.mark.parametrize("name", ["cfg1b", "cfg1b-rank1", "cfg3", "random-g"])
def test_strategy_modes_bitexact(name):
    """NEXT-2 dispatch strategies on the GPU equal the oracle path by path: physical (bid-curve) dispatch
    with recorded actions, self-scheduled at the lagged price, and a fixed schedule settled at the
    realised prices."""
    import torch
    if name == "cfg3":
        base = workloads.cfg2(T=2, K=2)
        inst = workloads.cfg3_gpu(oracle.actions(to_oracle(base)), T=20, K=12)
    elif name == "random-g":
        inst = workloads.random_instance(62, T=7, K=3, S_max=150)
        act = oracle.actions(to_oracle(inst))
        inst.payoff_kind = workloads.PAYOFF_LINEAR_MINUS_G
        inst.g = workloads.random_g(62, len(act), 3.0)
    else:
        inst = workloads.cfg1("b", rank1=name.endswith("rank1"))
        inst.s0 = inst.sbar * 0.5 + 0.3 * inst.delta
    pr = to_oracle(inst)
    ref = oracle.backward(pr)
    n = 1500
    with _gpu(inst) as s:
        s.backward()
        out = torch.empty(n, dtype=torch.float64, device="cuda")
        acts = torch.empty(inst.T * n, dtype=torch.int16, device="cuda")
        for mode, omode in ((E.ESDP_SIM_PHYSICAL, oracle.SIM_PHYSICAL), (E.ESDP_SIM_SELF, oracle.SIM_SELF)):
            want, wact = oracle.simulate_strategy(pr, ref.W, omode, n, seed=17, want_actions=True)
            E.esdp_simulate_strategy_dev(s.ctx, n, 17, mode, out.data_ptr(), actions_ptr=acts.data_ptr())
            torch.cuda.synchronize()
            assert np.array_equal(out.cpu().numpy(), want), mode
            assert np.array_equal(acts.cpu().numpy().reshape(inst.T, n), wact), mode
        sched = wact[:, 3].copy()
        want, _ = oracle.simulate_strategy(pr, None, oracle.SIM_FIXED, n, seed=17, schedule=sched)
        sd = torch.from_numpy(sched).cuda()
        E.esdp_simulate_strategy_dev(s.ctx, n, 17, E.ESDP_SIM_FIXED, out.data_ptr(), schedule_ptr=sd.data_ptr())
        torch.cuda.synchronize()
        assert np.array_equal(out.cpu().numpy(), want)


def test_price_paths_and_perfect_foresight():
    """esdp_price_paths_dev returns the realised prices of the simulation's paths (a constant schedule
    settles to p times their running sum, bit for bit); one context with K = n paths and identity
    transitions then solves every path's deterministic (perfect-foresight) DP, equal to the oracle's K = 1
    solve of that path."""
    import torch
    inst = workloads.cfg1("b")
    pr = to_oracle(inst)
    n = 12
    with _gpu(inst) as s:
        s.backward()
        lamp = torch.empty(inst.T * n, dtype=torch.float64, device="cuda")
        E.esdp_price_paths_dev(s.ctx, n, 23, lambda_ptr=lamp.data_ptr())
        act = s.actions()
        a = int(np.argmax(act))                                   # a constant schedule of the top power
        sd = torch.full((inst.T,), a, dtype=torch.int16, device="cuda")
        out = torch.empty(n, dtype=torch.float64, device="cuda")
        E.esdp_simulate_strategy_dev(s.ctx, n, 23, E.ESDP_SIM_FIXED, out.data_ptr(), schedule_ptr=sd.data_ptr())
        torch.cuda.synchronize()
        lam = lamp.cpu().numpy().reshape(inst.T, n)
        got = out.cpu().numpy()
    for j in range(n):
        acc = 0.0
        for t in range(inst.T):
            acc = acc + lam[t, j] * act[a]
        assert got[j] == acc
    # perfect foresight: K = n deterministic paths, identity transitions
    pf = workloads.Instance("pf", inst.T, n, inst.pbar, inst.sbar, inst.s0, inst.eta_c, inst.eta_d, inst.delta,
                            lam.copy(), np.broadcast_to(np.eye(n), (inst.T - 1, n, n)).copy(), np.full(n, 1.0 / n))
    with _gpu(pf) as s:
        s.backward()
        V1, _ = s.values(1)
    i0 = int(round(inst.s0 / inst.delta))
    for j in range(n):
        one = workloads.Instance("pf1", inst.T, 1, inst.pbar, inst.sbar, inst.s0, inst.eta_c, inst.eta_d, inst.delta,
                                 lam[:, j:j + 1].copy(), np.ones((inst.T - 1, 1, 1)), np.array([1.0]))
        assert V1[j, i0] == oracle.backward(to_oracle(one)).J


def test_lambda_only_load_after_side_stream_simulation():
    """a time-varying chain with more than 4096 distinct P_t rows builds its sampling
    tables lazily on the simulation's stream; a later lambda-only load copies those tables into the
    other input slot and must wait for that build.  Simulate on a side stream, load lambda only, and
    check that the next solve and simulation still equal the oracle bit for bit."""
    import dataclasses
    import torch
    x = workloads.cfg2(T=80, K=64)
    rng = np.random.Generator(np.random.PCG64(31337))
    P = rng.dirichlet(np.ones(x.K) * 0.3, size=(x.T - 1, x.K))     # 79 distinct slices, 5056 rows
    x = dataclasses.replace(x, P=np.ascontiguousarray(P))
    y = dataclasses.replace(x, lam=np.ascontiguousarray(x.lam * 1.25 + 3.0))
    rx = oracle.backward(to_oracle(x), nthreads=16)
    ry = oracle.backward(to_oracle(y), nthreads=16)
    n = 8192
    sx = oracle.simulate(to_oracle(x), rx.pol, n, seed=9)[0]
    sy = oracle.simulate(to_oracle(y), ry.pol, n, seed=9)[0]
    side = torch.cuda.Stream()
    out = torch.empty(n, dtype=torch.float64, device="cuda")
    with E.Solver(x) as s:
        assert s.backward() == rx.J
        E.esdp_simulate_dev(s.ctx, n, 9, out.data_ptr(), stream=side)   # lazy table build on `side`
        E.esdp_load(s.ctx, lam=y.lam)                                   # copies the old slot's tables
        side.synchronize()
        assert np.array_equal(out.cpu().numpy(), sx)
        assert s.backward() == ry.J
        E.esdp_simulate_dev(s.ctx, n, 9, out.data_ptr(), stream=side)
        side.synchronize()
        assert np.array_equal(out.cpu().numpy(), sy)
        per, _, _ = s.simulate(n, seed=9)
        assert np.array_equal(per, sy)


@pytest.mark.parametrize("rank1", [False, True])
def test_partial_loads_alternate_slots(rank1):
    """Loads that replace one array at a time (lambda only, g only, pi only, P only) alternate between the two
    input slots: a kept array is copied into the other slot only when that slot does not already hold it
    (upload generations), the sampling tables are built lazily by the next simulation.  After every load the
    solve, every policy and a simulation equal the oracle's on the combined inputs, bit for bit (LINEAR_MINUS_G
    payoff, so g and its window fit travel too)."""
    import dataclasses
    with E.Solver(workloads.cfg2(T=2, K=2)) as s0:
        acts = s0.actions()
    x = workloads.cfg3_gpu(acts, T=24, K=12, rank1=rank1)
    rng = np.random.Generator(np.random.PCG64(4242))
    lam2 = np.ascontiguousarray(x.lam * 1.1 - 2.0)
    g2 = np.ascontiguousarray(x.g * 0.5)
    if rank1:
        pi2 = rng.dirichlet(np.ones(x.K), size=x.T)
    else:
        pi2 = rng.dirichlet(np.ones(x.K))
    P2 = None if rank1 else np.ascontiguousarray(rng.dirichlet(np.ones(x.K) * 0.5, size=(x.T - 1, x.K)))
    steps = [dict(lam=lam2), dict(g=g2), dict(lam=x.lam), dict(pi=pi2), dict(P=P2), dict(lam=lam2), dict()]
    cur = dict(lam=x.lam, g=x.g, pi=x.pi, P=x.P)
    n = 4096
    with E.Solver(x) as s:
        for j, upd in enumerate(steps):
            upd = {k: v for k, v in upd.items() if v is not None}
            if upd:
                E.esdp_load(s.ctx, **upd)
            cur.update(upd)
            y = dataclasses.replace(x, **cur)
            pr = to_oracle(y)
            ref = oracle.backward(pr, nthreads=16)
            assert s.backward() == ref.J, j
            for t in (1, y.T // 2, y.T):
                assert np.array_equal(s.policy(t), ref.pol[t - 1]), (j, t)
            per, _, _ = s.simulate(n, seed=11 + j)
            assert np.array_equal(per, oracle.simulate(pr, ref.pol, n, seed=11 + j)[0]), j


@pytest.mark.parametrize("name", ["cfg2-small", "cfg2-rank1-small"])
def test_dmma_probe_failure_falls_back_to_dfma(name, monkeypatch):
    """The DMMA bit-exactness guard: a failed DMMA-vs-fma-chain probe at context creation (forced with
    ESDP_DMMA_PROBE_FAIL=1) moves the expectation to DFMA; the plan reports it and every result is still the
    oracle's, bit for bit (single and batch contexts).  Without the variable the probe passes on B200."""
    inst = workloads.cfg2(T=12, K=24, rank1=name.endswith("rank1-small"))
    pr = to_oracle(inst)
    ref = oracle.backward(pr, nthreads=8)
    with E.Solver(inst) as s:
        assert s.stencil_kind & 2 and not s.stencil_kind & 4
    monkeypatch.setenv("ESDP_DMMA_PROBE_FAIL", "1")
    with E.Solver(inst) as s:
        assert s.stencil_kind & 4 and not s.stencil_kind & 2
        assert s.backward() == ref.J
        for t in range(1, inst.T + 1):
            V, W = s.values(t)
            assert np.array_equal(V, ref.V[t - 1]) and np.array_equal(W, ref.W[t - 1])
            assert np.array_equal(s.policy(t), ref.pol[t - 1])


@pytest.mark.parametrize("generic", ["0", "1"])
@pytest.mark.parametrize("force_nonuni", ["0", "1"])
@pytest.mark.parametrize("opt", ["1", "2", "4"])
def test_window_kernel_variants(opt, force_nonuni, generic, monkeypatch):
    """Every window-stencil variant gives the oracle's bits: one, two or four outputs per thread
    (ESDP_WIN_OPT; four is the throughput-regime default), the Eq. 10 fast query path or the generic one
    (ESDP_WIN_GENERIC=1), and the non-unimodal fallbacks forced on every table (ESDP_WIN_FORCE_NONUNI=1): the
    raw-key window scan (linear payoff) and the packed sparse tables (payoff lambda p - g).  Ragged tails (S
    not a multiple of the tile), several tiles, T > 2."""
    if generic == "1" and force_nonuni == "1":
        pytest.skip("the non-unimodal fallbacks never take the fast path")
    monkeypatch.setenv("ESDP_WIN_OPT", opt)
    monkeypatch.setenv("ESDP_WIN_FORCE_NONUNI", force_nonuni)
    monkeypatch.setenv("ESDP_WIN_GENERIC", generic)
    for inst in (workloads.cfg2(T=5, K=12), workloads.cfg1("b"), workloads.random_instance(77, T=4, K=3, S_max=900)):
        _compare_all(inst, nthreads=16, expect_window=True)
    base = workloads.cfg2(T=2, K=2)
    _compare_all(workloads.cfg3_gpu(oracle.actions(to_oracle(base)), T=5, K=8), nthreads=16, expect_window=True)
