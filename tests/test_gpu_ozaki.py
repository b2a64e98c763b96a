"""NEXT-4: the expectation W = P V (Alg. 1 line 11; Eq. 6) as Ozaki-sliced u8
products on the 5th-generation tensor cores (tcgen05.mma kind::i8, ozaki.cuh).  This path is NOT the
canonical fma chain (R15), so its bar is north_star's tolerance instead of bit equality:

* the product itself against an extended-precision reference (numpy longdouble, 64-bit mantissa): every
  entry within the error bound of ozaki.cuh, 4 (2 K 2^-64 + 64 2^-80) max_k' P[m][k'] max_k' V[k'][n], plus
  the final rounding -- at full cfg5 width and on ragged shapes;
* a whole batch backward on the Ozaki plan against the FP64 oracle: J and V_1 within 1e-9 relative
  (north_star; the measured error is ~1e-14), and every policy entry equal to the oracle's except at
  documented ties: the oracle's own candidates of the two actions differ by <= 1e-10 relative
  (SURVEY §8(c).4)."""
import numpy as np
import pytest
import torch

import oracle
import workloads
from helpers import to_oracle

pytestmark = pytest.mark.gpu

import paper_2511_15629_b200 as E  # no skip: a missing library must fail loudly


def _operands(rows, K, ncols, ldv, seed):
    rng = np.random.default_rng(seed)
    P = rng.random((rows, K)) ** 6                      # wide dynamic range inside a row, tiny entries
    P[:, rng.random(K) < 0.1] = 0.0
    P /= np.maximum(P.sum(axis=1, keepdims=True), 1e-300)
    scale = 10.0 ** rng.integers(-3, 7, size=ncols)     # columns of very different magnitude
    V = np.zeros((K, ldv))
    V[:, :ncols] = rng.random((K, ncols)) * scale
    Vc = V[:, :ncols]                                   # a view
    Vc[:, rng.random(ncols) < 0.05] = 0.0               # all-zero columns
    Vc[rng.random((K, ncols)) < 0.02] = 0.0
    return P, V


def _run(P, V, rows, K, ncols, ldv, ldw, method):
    dev = torch.device("cuda")
    Pd = torch.from_numpy(np.ascontiguousarray(P)).to(dev)
    Vd = torch.from_numpy(np.ascontiguousarray(V)).to(dev)
    Wd = torch.full((rows, ldw), np.nan, dtype=torch.float64, device=dev)
    E.expectation_dev(Pd.data_ptr(), Vd.data_ptr(), Wd.data_ptr(), rows, K, ncols, ldv, ldw, method)
    torch.cuda.synchronize()
    return Wd.cpu().numpy()


@pytest.mark.parametrize("rows,K,ncols,ldv,ldw", [(100, 100, 1001, 1004, 1004), (128, 128, 64, 64, 72), (8, 12, 33, 40, 33),
                                                  (1, 1, 1, 4, 1), (100, 100, 128512, 128512, 128512),
                                                  (57, 100, 2049, 2052, 2060)])
def test_ozaki_product_error_bound(rows, K, ncols, ldv, ldw):
    P, V = _operands(rows, K, ncols, ldv, seed=rows * 7919 + K * 31 + ncols)
    W = _run(P, V, rows, K, ncols, ldv, ldw, method=1)
    ex = P.astype(np.longdouble) @ V[:, :ncols].astype(np.longdouble)
    bound = 4.0 * (2 * K * 2.0 ** -64 + 64 * 2.0 ** -80) * np.outer(P.max(axis=1), V[:, :ncols].max(axis=0))
    err = np.abs(W[:, :ncols].astype(np.longdouble) - ex)
    # + the final FP64 rounding, + the reference's own error (longdouble, 64-bit mantissa)
    assert np.all(err <= bound + 2.0 ** -52 * np.abs(ex) + K * 2.0 ** -63 * np.abs(ex)), float(np.max(err / (bound + 1e-300)))
    assert np.all(np.isnan(W[:, ncols:])), "columns past ncols must stay untouched"
    # the canonical path (method 0) on the same operands is within the textbook bound K u sum |P||V|
    if ldv == ldw:
        W0 = _run(P, V, rows, K, ncols, ldv, ldw, method=0)
        err0 = np.abs(W0[:, :ncols].astype(np.longdouble) - ex)
        assert np.all(err0 <= K * 2.0 ** -53 * (P.astype(np.longdouble) @ V[:, :ncols].astype(np.longdouble)) + 1e-300)


def test_expectation_dev_rejects_bad_arguments():
    dev = torch.device("cuda")
    x = torch.zeros(16, dtype=torch.float64, device=dev)
    p = x.data_ptr()
    for args in [(0, 4, 4, 4, 4, 1), (4, 4, 8, 4, 4, 1), (200, 4, 4, 4, 4, 1), (4, 200, 4, 4, 4, 1), (4, 4, 4, 4, 8, 0),
                 (4, 4, 4, 4, 4, 7)]:
        with pytest.raises(E.EsdpError) as ei:
            E.expectation_dev(p, p, p, *args)
        assert ei.value.status == E.ESDP_E_CONFIG


def _cands(pr, tb, acts, lam, W_row, i):
    """The oracle's candidates fl(fl(lambda p_a) + Wint(i, a)) of every feasible action at row i (R14)."""
    out = np.full(len(acts), -np.inf)
    for a in range(len(acts)):
        if not (tb["ilo"][a] <= i <= tb["ihi"][a]):
            continue
        j = i + tb["off"][a]
        wint = W_row[j] if tb["w"][a] == 0.0 else tb["omw"][a] * W_row[j] + tb["w"][a] * W_row[j + 1]
        out[a] = lam * acts[a] + wint
    return out


def test_batch_ozaki_plan_within_tolerance():
    """cfg5 storage configurations on a cfg2 price chain (K = 100) on the Ozaki plan: J and V_1 within 1e-9
    relative of the oracle, every policy difference a documented tie."""
    idx = [0, 300, 777, 1023]
    insts = workloads.cfg5_instances(idx, T=10, K=100)
    with E.Batch(insts, ozaki=True) as b:
        assert b.plan == 2
        J = b.backward()
        worst = 0.0
        ties = 0
        for m, inst in enumerate(insts):
            pr = to_oracle(inst)
            ref = oracle.backward(pr, nthreads=16)
            assert abs(J[m] - ref.J) <= 1e-9 * abs(ref.J), (m, J[m], ref.J)
            V1 = b.value1(m)
            rel = np.max(np.abs(V1 - ref.V[0]) / np.maximum(1.0, np.abs(ref.V[0])))
            assert rel <= 1e-9, (m, rel)
            worst = max(worst, rel, abs(J[m] - ref.J) / abs(ref.J))
            acts = oracle.actions(pr)
            tb = oracle.tables(pr)
            for t in range(1, inst.T + 1):
                pol = b.policy(m, t)
                bad = np.argwhere(pol != ref.pol[t - 1])
                for k, i in bad:
                    c = _cands(pr, tb, acts, inst.lam[t - 1, k], ref.W[t - 1][k], i)
                    ag, ao = int(pol[k, i]), int(ref.pol[t - 1][k, i])
                    assert np.isfinite(c[ag]), (m, t, k, i, ag)   # the GPU's action is feasible
                    assert abs(c[ag] - c[ao]) <= 1e-10 * max(1.0, abs(ref.V[t - 1][k, i])), (m, t, k, i, c[ag], c[ao])
                    ties += 1
        print(f"Ozaki plan: worst relative error of J / V_1 {worst:.2e}, documented policy ties {ties}")
        assert worst < 1e-11   # the measured error is ~1e-14: a regression to a coarser product fails here
    with E.Batch(insts) as b:   # without the flag the batch keeps the canonical DMMA plan
        assert b.plan == 0


def test_ozaki_flag_ignored_where_it_does_not_apply():
    """K > 128 (cfg4 shape) or a zero action with a negative payoff (g(0) > 0: V may be negative) keep the
    canonical plan; rank-1 batches too."""
    insts = workloads.cfg5_instances([0, 1023], T=4, K=130)
    with E.Batch(insts, ozaki=True) as b:
        assert b.plan == 0
    base = workloads.cfg5_instances([5], T=4, K=8)[0]
    with E.Solver(workloads.cfg2(T=2, K=2)) as s0:
        acts = s0.actions()
    g = workloads.degradation_g(acts)
    g[np.argmin(np.abs(acts))] = 1.0          # payoff of the zero action -1 < 0
    inst = workloads.cfg3_gpu(acts, T=4, K=8)
    inst.g = g
    with E.Batch([inst], ozaki=True) as b:
        assert b.plan == 0
    inst.g = workloads.degradation_g(acts)    # g(0) = 0: granted
    with E.Batch([inst], ozaki=True) as b:
        assert b.plan == 2
    del base
