"""GPU parity of batch contexts (esdp_create_batch, cfg5): every instance of a batch -- one graph, one
expectation launch over the stacked values and one window launch over all instances per stage -- is
bit-identical to the oracle on that instance alone (J, V_1, every policy), and its simulated paths are
those of a context of its own."""
import numpy as np
import pytest

import oracle
import workloads
from helpers import to_oracle

pytestmark = pytest.mark.gpu

import paper_2511_15629_b200 as E  # no skip: a missing library must fail loudly


def _check_batch(insts, nthreads=16):
    with E.Batch(insts) as b:
        J = b.backward()
        for m, inst in enumerate(insts):
            ref = oracle.backward(to_oracle(inst), nthreads=nthreads)
            assert J[m] == ref.J, (m, J[m], ref.J)
            assert np.array_equal(b.value1(m), ref.V[0]), m
            for t in range(1, inst.T + 1):
                assert np.array_equal(b.policy(m, t), ref.pol[t - 1]), (m, t)
        J2 = b.backward()
        assert np.array_equal(J, J2)
        return b.A


@pytest.mark.parametrize("rank1", [False, True])
def test_batch_cfg5_sample(rank1):
    """Six cfg5 storage configurations (different pbar/delta, eta -> different action grids) on a short
    cfg2 price chain."""
    idx = [0, 37, 300, 511, 777, 1023]
    insts = workloads.cfg5_instances(idx, T=12, K=10)
    if rank1:
        base = workloads.cfg2(T=12, K=10, rank1=True)
        for x in insts:
            x.P, x.pi = None, base.pi
            x.lam = base.lam
    A = _check_batch(insts)
    assert len(set(A)) > 1


def test_batch_mixed_plans_and_payoffs():
    """A batch mixing window-plan instances, a brute-force instance (too few actions per side), an
    affine degradation payoff (window) and a non-affine one (brute), plus an off-grid s0."""
    base = workloads.cfg1("b")
    insts = []
    for j, (pbar, eta, s0) in enumerate([(9.5, 0.9, 0.0), (1.5, 0.95, 50.0), (20.0, 0.85, 33.3), (9.5, 0.9, 10.0)]):
        x = workloads.Instance(f"mix{j}", base.T, base.K, pbar, base.sbar, s0, eta, eta, base.delta, base.lam, base.P,
                               base.pi)
        insts.append(x)
    act3 = oracle.actions(to_oracle(insts[3]))
    insts[3].payoff_kind = workloads.PAYOFF_LINEAR_MINUS_G
    insts[3].g = 2.0 * np.abs(act3) + 5.0 * (act3 != 0)
    act0 = oracle.actions(to_oracle(insts[0]))
    insts[0].payoff_kind = workloads.PAYOFF_LINEAR_MINUS_G
    insts[0].g = workloads.random_g(3, len(act0), 4.0)
    _check_batch(insts)


def test_batch_simulation_matches_single_contexts():
    import torch
    insts = workloads.cfg5_instances([5, 400, 900], T=16, K=12)
    n_paths = 3000
    with E.Batch(insts) as b:
        b.backward()
        out = torch.zeros(len(insts) * n_paths, dtype=torch.float64, device="cuda")
        b.simulate_dev(n_paths, 77, out.data_ptr())
        torch.cuda.synchronize()
        got = out.cpu().numpy().reshape(len(insts), n_paths)
    for m, inst in enumerate(insts):
        with E.Solver(inst, keep_values=False) as s:
            s.backward()
            per, _, _ = s.simulate(n_paths, seed=77 + m)
        assert np.array_equal(got[m], per), m


def test_batch_rejects_mismatched_price_models():
    a, b = workloads.cfg5_instances([1, 2], T=6, K=5)
    b.lam = b.lam + 1.0
    with pytest.raises(E.EsdpError) as e:
        E.Batch([a, b])
    assert e.value.status == E.ESDP_E_CONFIG
    c = workloads.cfg5_instances([3], T=6, K=5)[0]
    c.payoff_kind = workloads.PAYOFF_TABLE
    c.g = np.zeros((6, 5, 10))
    with pytest.raises(E.EsdpError) as e:
        E.Batch([a, c])
    assert e.value.status == E.ESDP_E_CONFIG


def test_batch_full_horizon_cfg5():
    """Four cfg5 configurations at full cfg2 size (T=288, S=1001, K=100) in one batch: J, V_1 and the
    policies of sampled stages bit-identical to the oracle on each instance."""
    insts = workloads.cfg5_instances([0, 341, 682, 1023])
    with E.Batch(insts) as b:
        J = b.backward()
        for m, inst in enumerate(insts):
            ref = oracle.backward(to_oracle(inst), nthreads=16)
            assert J[m] == ref.J
            assert np.array_equal(b.value1(m), ref.V[0])
            for t in (1, 100, 287, 288):
                assert np.array_equal(b.policy(m, t), ref.pol[t - 1]), (m, t)


@pytest.mark.parametrize("rank1", [False, True])
def test_batch_load_async_replaces_price_model(rank1):
    """esdp_batch_load_async: a batch built on one price model and reloaded with another (validated, copied
    on the stream, sampling tables rebuilt) solves the new model bit for bit -- J, V_1, the policies and
    the simulated paths equal those of a batch created on the new model."""
    import torch
    idx = [5, 300, 900]
    a = workloads.cfg5_instances(idx, T=12, K=12)
    b = workloads.cfg5_instances(idx, T=12, K=12)
    lam_b, P_b, _ = workloads.price_chain(12, 12, 5.0 / 60.0, seed=workloads.SEED_BASE + 99)
    rng = np.random.default_rng(3)   # another time-homogeneous chain (one distinct slice, as a's)
    P0 = P_b[0] * rng.uniform(0.5, 1.5, P_b[0].shape)
    P_b = np.ascontiguousarray(np.broadcast_to(P0 / P0.sum(axis=1, keepdims=True), P_b.shape))
    for x in b:
        x.lam, x.P = lam_b, P_b
    if rank1:
        base = workloads.cfg2(T=12, K=12, rank1=True)
        for x in a:
            x.P, x.pi = None, base.pi
        for x in b:
            x.P, x.pi = None, base.pi
    s = torch.cuda.Stream()
    out1 = torch.zeros(len(idx) * 256, dtype=torch.float64, device="cuda")
    out2 = torch.zeros_like(out1)
    with E.Batch(b) as ref:
        Jr = ref.backward()
        ref.simulate_dev(256, 7, out2.data_ptr())
        torch.cuda.synchronize()
        pols = [[ref.policy(m, t) for t in range(1, 13)] for m in range(len(idx))]
        V1 = [ref.value1(m) for m in range(len(idx))]
    with E.Batch(a) as bt:
        bt.backward()
        lam = np.ascontiguousarray(b[0].lam)
        P = None if rank1 else np.ascontiguousarray(b[0].P)
        pi = np.ascontiguousarray(b[0].pi)
        bt.load_async(lam.ctypes.data, None if P is None else P.ctypes.data, pi.ctypes.data, s)
        bt.backward_async(s)
        bt.simulate_dev(256, 7, out1.data_ptr(), s)
        s.synchronize()
        assert np.array_equal(bt.objective(), Jr)
        for m in range(len(idx)):
            assert np.array_equal(bt.value1(m), V1[m])
            for t in range(1, 13):
                assert np.array_equal(bt.policy(m, t), pols[m][t - 1])
        assert torch.equal(out1, out2)
        bad = lam.copy()
        bad[0, 0] = np.nan
        with pytest.raises(E.EsdpError):
            bt.load_async(bad.ctypes.data, None if P is None else P.ctypes.data, pi.ctypes.data, s)


def test_batch_kernel_times():
    """esdp_batch_kernel_time: the diagnostic per-launch times of the batch's stage kernels are positive."""
    with E.Batch(workloads.cfg5_instances([0, 512], T=6, K=8)) as bt:
        bt.backward()
        assert bt.kernel_time(0, 10) > 0 and bt.kernel_time(1, 10) > 0
        with pytest.raises(E.EsdpError):
            bt.kernel_time(2, 10)   # no brute-force instances in this batch


@pytest.mark.parametrize("generic", ["0", "1"])
@pytest.mark.parametrize("opt", ["1", "2", "4"])
def test_batch_window_variants(opt, generic, monkeypatch):
    """The batch window kernel with one, two or four outputs per thread (ESDP_WIN_OPT), on the Eq. 10 fast
    query path or forced onto the generic one (ESDP_WIN_GENERIC=1), gives the same bits."""
    monkeypatch.setenv("ESDP_WIN_OPT", opt)
    monkeypatch.setenv("ESDP_WIN_GENERIC", generic)
    _check_batch(workloads.cfg5_instances([0, 37, 300, 1023], T=8, K=10))


@pytest.mark.parametrize("pres", ["1", "0"])
def test_batch_wide_expectation_tiling(pres, monkeypatch):
    """48 cfg5 configurations (K = 100: 4.8e6 expectation outputs per stage, >= 4e6) take the P-resident
    persistent expectation (default: P_t kept in shared memory, 64-column V tiles double-buffered) or, with
    ESDP_PRES=0, the wide DMMA tiling (16 x 128 blocks, two stages): every instance bit-identical to the
    oracle either way; also in two instance groups of 48 and 49 configurations (each group's product
    >= 4e6 outputs, at a column offset)."""
    monkeypatch.setenv("ESDP_PRES", pres)
    idx = [(j * 1024) // 48 for j in range(48)]
    _check_batch(workloads.cfg5_instances(idx, T=3, K=100))
    monkeypatch.setenv("ESDP_BATCH_GROUPS", "2")
    idx = [(j * 1024) // 97 for j in range(97)]
    _check_batch(workloads.cfg5_instances(idx, T=2, K=100))


@pytest.mark.parametrize("groups", ["1", "2", "3"])
def test_batch_instance_groups(groups, monkeypatch):
    """Instance groups with independent stage chains (graph branches; the default from 128 instances on):
    every instance bit-identical to the oracle for 1, 2 and 3 groups of a 9-instance batch (ragged groups)."""
    monkeypatch.setenv("ESDP_BATCH_GROUPS", groups)
    idx = [0, 37, 100, 300, 511, 640, 777, 900, 1023]
    _check_batch(workloads.cfg5_instances(idx, T=10, K=12))


def test_batch_plan_reports_the_dfma_fallback(monkeypatch):
    """esdp_batch_plan: 0 (FP64 DMMA) by default; 1 (DFMA) when the DMMA bit-exactness probe fails (forced with
    ESDP_DMMA_PROBE_FAIL=1), and every instance is still the oracle's, bit for bit."""
    insts = workloads.cfg5_instances([0, 600], T=5, K=12)
    with E.Batch(insts) as b:
        assert b.plan == 0
    monkeypatch.setenv("ESDP_DMMA_PROBE_FAIL", "1")
    with E.Batch(insts) as b:
        assert b.plan == 1
    _check_batch(insts)
