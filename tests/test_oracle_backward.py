"""Pins of the oracle's backward induction (Alg. 1 lines 6-11, Eqs. 5-6).

Each test checks the oracle against something other than itself: SPEC worked examples,
closed forms, exact-rational brute force, enumeration of all action sequences, the LP/MILP
optimum of Eqs. 1/3 (scipy HiGHS), a literal transliteration of Algorithm 1, symmetries and
invariants."""
import dataclasses
import math
from fractions import Fraction

import numpy as np
import pytest

import oracle
import pins
import workloads
from helpers import to_oracle, simple_problem


def _solve(pr, **kw):
    return oracle.backward(pr, **kw)


# --- SPEC worked examples (tests/golden/spec_examples.txt) -----------------------------------

def test_spec_dp_examples():
    """S:249-251 (dp1-dp3)."""
    sol = _solve(simple_problem(1.0, 1.0, 0.5, 1.0, lam=[10.0]))
    assert sol.V[0, 0].tolist() == [0.0, 5.0, 10.0]
    sol = _solve(simple_problem(1.0, 1.0, 0.5, 1.0, lam=[-5.0]))
    assert sol.V[0, 0].tolist() == [5.0, 2.5, 0.0]
    sol = _solve(simple_problem(1.0, 1.0, 0.5, 1.0, T=3, K=2, lam=np.zeros((3, 2))))
    assert np.all(sol.V == 0.0) and np.all(sol.W == 0.0)


def test_two_price_arbitrage_closed_form():
    """dp4 (S:262 corrected, R21): prices [-1, 2], s0 = 0, eta = 1: Eq. 1 optimum = 1*1 + 2*1 = 3."""
    sol = _solve(simple_problem(1.0, 1.0, 0.5, 1.0, T=2, lam=[-1.0, 2.0], s0=0.0))
    assert sol.J == 3.0
    v = pins.enumerate_sequences([-1.0, 2.0], [-1, -0.5, 0, 0.5, 1], 1.0, 0.0, 1.0, 1.0)
    assert v == 3.0


def test_equal_prices_lossy_is_zero():
    """dp5: with eta < 1, constant prices make every round trip lose money -> 0 from s0 = 0."""
    pr = simple_problem(1.0, 4.0, 0.1, math.sqrt(0.85), T=6, lam=[7.0] * 6, s0=0.0)
    assert _solve(pr).J == 0.0


def test_single_high_price_full_battery():
    """dp6: prices [5], s0 = sbar (and sbar*eta >= pbar) -> discharge pbar: J = 5 pbar."""
    pr = simple_problem(1.0, 4.0, 0.5, 1.0, T=1, lam=[5.0], s0=4.0)
    assert _solve(pr).J == 5.0


# --- brute force on tiny inputs --------------------------------------------------------------

@pytest.mark.parametrize("seed", range(30))
def test_exact_rational_expectimax(seed):
    """V7: grid-MDP expectimax in exact rational arithmetic (top-down recursion, lottery at off-grid
    endpoints) equals the FP64 oracle to 1e-12 relative, for J and for every V_1(i, k)."""
    inst = workloads.random_instance(seed, T=None, K=None, S_max=8)
    pr = to_oracle(inst)
    act = oracle.actions(pr)
    sol = _solve(pr)
    J_exact, Vk = pins.expectimax_exact(inst, act)
    assert abs(sol.J - float(J_exact)) <= 1e-12 * max(1.0, abs(float(J_exact)))
    for k in range(inst.K):
        for i in range(inst.S):
            ex = float(Vk(1, i, k))
            assert abs(sol.V[0, k, i] - ex) <= 1e-12 * max(1.0, abs(ex)), (seed, k, i)


@pytest.mark.parametrize("seed", range(12))
def test_exact_rational_expectimax_general_payoff(seed):
    """V7 with the non-concave payoff lambda p - g(p) and with a full payoff table (D3)."""
    kind = workloads.PAYOFF_LINEAR_MINUS_G if seed % 2 == 0 else workloads.PAYOFF_TABLE
    inst = workloads.random_instance(seed + 100, S_max=7)
    pr = to_oracle(inst)
    S, A = oracle.dims(pr)
    act = oracle.actions(pr)
    if kind == workloads.PAYOFF_LINEAR_MINUS_G:
        g = workloads.random_g(seed, A)
        pay = lambda t, k, a: Fraction(inst.lam[t - 1][k]) * Fraction(act[a]) - Fraction(g[a])
    else:
        g = workloads.random_table(seed, inst.T, inst.K, A)
        pay = lambda t, k, a: Fraction(g[t - 1][k][a])
    inst.payoff_kind, inst.g = kind, g
    pr = to_oracle(inst)
    sol = _solve(pr)
    J_exact, _ = pins.expectimax_exact(inst, act, payoff=pay)
    assert abs(sol.J - float(J_exact)) <= 1e-12 * max(1.0, abs(float(J_exact)))


@pytest.mark.parametrize("seed", range(15))
def test_enumerate_all_action_sequences(seed):
    """north_star: brute-force enumeration of all action sequences for T <= 6 (K = 1, on-lattice
    so the continuous SoC path stays on the grid, R16)."""
    rng = np.random.default_rng(seed)
    T = int(rng.integers(1, 7))
    inst = workloads.random_instance(seed + 500, T=T, K=1, S_max=6, lattice=True, rank1=False)
    pr = to_oracle(inst)
    act = oracle.actions(pr)
    if len(act) ** T > 2e5:
        pytest.skip("enumeration too large")
    sol = _solve(pr)
    v = pins.enumerate_sequences(inst.lam[:, 0], act, inst.sbar, inst.s0, 1.0, 1.0)
    assert abs(sol.J - v) <= 1e-12 * max(1.0, abs(v))


# --- LP / MILP (Eqs. 1 and 3), scipy HiGHS ---------------------------------------------------

@pytest.mark.parametrize("seed", range(4))
def test_deterministic_dp_equals_lp_on_lattice(seed):
    """V8: K=1, eta=1, pbar, sbar, s0 on the delta lattice: the LP of Eq. 1 has an integral optimal
    vertex (difference constraints are totally unimodular), so DP = LP."""
    rng = np.random.default_rng(seed)
    T = 48
    lam = rng.normal(40.0, 15.0, size=(T, 1))
    pr = simple_problem(3.0, 12.0, 1.0, 1.0, T=T, lam=lam, s0=float(rng.integers(0, 13)))
    J = _solve(pr).J
    lp, _ = pins.lp_value(lam[:, 0], 3.0, 12.0, pr.s0, 1.0, 1.0)
    assert abs(J - lp) <= 1e-9 * abs(lp)


def test_dp_below_lp_gap_shrinks_with_delta():
    """V9 / Table 1 trend: with eta < 1 and lambda >= 0 the DP is a restriction (<= LP), and
    the gap shrinks as delta is refined."""
    rng = np.random.default_rng(7)
    T = 72
    lam = np.abs(rng.normal(40.0, 15.0, size=(T, 1))) + 40 * np.sin(np.arange(T) * 2 * np.pi / 24)[:, None] ** 2
    eta = math.sqrt(0.85)
    lp, _ = pins.lp_value(lam[:, 0], 1.0, 4.0, 0.0, eta, eta)
    gaps = []
    for d in [0.1, 0.05, 0.02]:
        J = _solve(simple_problem(1.0, 4.0, d, eta, T=T, lam=lam)).J
        assert J <= lp + 1e-9
        gaps.append((lp - J) / lp)
    assert gaps[0] > gaps[1] > gaps[2] >= 0.0
    assert gaps[0] < 0.02


def test_negative_prices_table2_structure():
    """V10 / Table 2: K=1, all lambda <= 0, s0 = sbar: LP relaxation >= MILP >= DP,
    the LP restriction (no discharge at lambda <= 0) earns exactly 0, and the DP is
    within a few tenths of a percent of the MILP."""
    inst = workloads.cfg3_small()
    pr = to_oracle(inst)
    J = _solve(pr).J
    lam = inst.lam[:, 0]
    relax, compl = pins.lp_value(lam, inst.pbar, inst.sbar, inst.s0, inst.eta_c, inst.eta_d)
    mip, mip_compl = pins.lp_value(lam, inst.pbar, inst.sbar, inst.s0, inst.eta_c, inst.eta_d, integer=True)
    restr, _ = pins.lp_value(lam, inst.pbar, inst.sbar, inst.s0, inst.eta_c, inst.eta_d, restrict_neg=True)
    assert relax >= mip - 1e-6 >= J - 2e-6
    assert abs(restr) < 1e-7
    assert mip_compl == 0 and compl > 0
    assert (mip - J) / mip < 0.01


# --- the paper's own algorithm (rank-1) -----------------------------------------------------

@pytest.mark.parametrize("variant", ["a", "b"])
def test_rank1_equals_literal_algorithm1(variant):
    """V11: with stagewise-independent prices (P_t = 1 pi_{t+1}^T) the Markov recursion is the
    paper's Algorithm 1; compare with a literal numpy transliteration (S x P x R tensor)."""
    inst = workloads.cfg1(variant, rank1=True)
    pr = to_oracle(inst)
    act = oracle.actions(pr)
    assert np.array_equal(act, pins.paper_actions(inst.pbar, inst.eta_c, inst.eta_d, inst.delta))
    sol = _solve(pr)
    V_hat = pins.alg1_numpy(inst, act)
    # our W_t == paper V_hat_t for t = 1..T-1, and sum_k pi_1[k] V_1[k] == paper V_hat_0
    for t in range(1, inst.T):
        np.testing.assert_allclose(sol.W[t - 1, 0], V_hat[t], rtol=1e-12, atol=1e-9)
        assert np.array_equal(sol.W[t - 1, 0], sol.W[t - 1, -1])   # identical across k (rank-1)
    V0 = inst.pi[0] @ sol.V[0]
    np.testing.assert_allclose(V0, V_hat[0], rtol=1e-12, atol=1e-9)


# --- symmetries and invariants ----------------------------------------------------------------

@pytest.mark.parametrize("seed", range(10))
def test_price_scaling_is_exact(seed):
    """V12: lambda -> 2 lambda (and g -> 2 g) doubles V exactly (scaling by 2 is exact in binary64)
    and keeps the policy."""
    inst = workloads.random_instance(seed + 40, S_max=20)
    pr = to_oracle(inst)
    S, A = oracle.dims(pr)
    inst.payoff_kind, inst.g = workloads.PAYOFF_LINEAR_MINUS_G, workloads.random_g(seed, A)
    a = _solve(to_oracle(inst))
    inst.lam = inst.lam * 2.0
    inst.g = inst.g * 2.0
    b = _solve(to_oracle(inst))
    assert np.array_equal(b.V, 2.0 * a.V) and np.array_equal(b.pol, a.pol)


@pytest.mark.parametrize("seed", range(10))
def test_mirror_symmetry_eta_one(seed):
    """V12: with eta = 1 the problem is symmetric under s -> sbar - s, lambda -> -lambda:
    V(s; lambda) == V(sbar - s; -lambda) exactly."""
    inst = workloads.random_instance(seed + 60, S_max=20, lattice=True)
    a = _solve(to_oracle(inst))
    inst.lam = -inst.lam
    b = _solve(to_oracle(inst))
    assert np.array_equal(a.V, b.V[:, :, ::-1])


@pytest.mark.parametrize("seed", range(20))
def test_invariants(seed):
    """V13 / R18: V >= 0; V_t >= W_t = P_t V_{t+1} (do-nothing is feasible); V_T = best one-shot
    payoff; every policy action is feasible; results independent of the thread count."""
    inst = workloads.random_instance(seed + 80, S_max=40, T=6, K=3)
    pr = to_oracle(inst)
    sol = _solve(pr)
    sol4 = _solve(pr, nthreads=4)
    assert np.array_equal(sol.V, sol4.V) and np.array_equal(sol.pol, sol4.pol)
    assert np.all(sol.V >= 0.0)
    assert np.all(sol.V >= sol.W)
    tb = oracle.tables(pr)
    act = oracle.actions(pr)
    S = inst.S
    for k in range(inst.K):
        for i in range(S):
            feas = [a for a in range(len(act)) if tb["ilo"][a] <= i <= tb["ihi"][a]]
            assert sol.V[-1, k, i] == max(inst.lam[-1, k] * act[a] for a in feas)
    ii = np.arange(S)[None, None, :]
    assert np.all((tb["ilo"][sol.pol] <= ii) & (ii <= tb["ihi"][sol.pol]))


@pytest.mark.parametrize("seed", range(12))
def test_policy_is_smallest_exact_argmax(seed):
    """R8: the policy is the smallest action index attaining the max.  Integer prices
    on an eta = 1 lattice make every candidate exact in binary64, so ties are exact; the smallest
    maximizer is computed independently from the exact-rational recursion."""
    rng = np.random.default_rng(seed)
    inst = workloads.random_instance(seed + 900, S_max=10, lattice=True, T=4)
    inst.lam = np.round(rng.normal(0.0, 3.0, size=inst.lam.shape))   # many exact ties
    pr = to_oracle(inst)
    act = oracle.actions(pr)
    sol = _solve(pr)
    pins.expectimax_exact(inst, act)
    ctx = pins.expectimax_exact.last
    EV, moves, pay = ctx["EV"], ctx["moves"], ctx["pay"]
    for t in range(1, inst.T + 1):
        for k in range(inst.K):
            for i in range(inst.S):
                cands = []
                for a, (o, w) in enumerate(moves):
                    assert w == 0
                    if 0 <= i + o <= inst.S - 1:
                        cands.append((pay(t, k, a) + EV(t, i + o, k), a))
                m = max(c for c, _ in cands)
                first = min(a for c, a in cands if c == m)
                assert sol.pol[t - 1, k, i] == first, (t, k, i)


def test_table1_year_trend():
    """NEXT-3 / Table 1: deterministic hourly year (T = 8784), 4-h battery, eta = sqrt(0.85):
    the DP is a restriction of the LP (DP <= LP), the gap shrinks as delta is refined through
    0.10 / 0.05 / 0.02 / 0.01 (A = 22 / 42 / 103 / 203), and is a small fraction of a percent at 0.01
    (paper: -0.19 / -0.13 / -0.04 / -0.02 %)."""
    inst = workloads.table1_deterministic(0.1)
    lp, _ = pins.lp_value(inst.lam[:, 0], 1.0, 4.0, 0.0, inst.eta_c, inst.eta_d)
    gaps = []
    for d, A in [(0.1, 22), (0.05, 42), (0.02, 103), (0.01, 203)]:
        inst = workloads.table1_deterministic(d)
        pr = to_oracle(inst)
        assert oracle.dims(pr)[1] == A
        J = _solve(pr, nthreads=8).J
        assert J <= lp + 1e-6
        gaps.append((lp - J) / lp)
    assert gaps[0] > gaps[1] > gaps[2] > gaps[3] > 0.0
    assert gaps[0] < 0.005 and gaps[3] < 0.001


# --- R24: off-grid s0 (Eq. 6 at t = 0; interpolation rule S:252-255) ------------------

@pytest.mark.parametrize("s0, J_closed", [(0.3, 3.0), (0.8, 8.0), (0.1, 1.0)])
def test_objective_off_grid_s0_closed_form(s0, J_closed):
    """T = 1, K = 1, eta = 1, lambda = 10, pbar = 1, delta = 0.5, sbar = 2: V_1 = [0, 5, 10, 10, 10]
    (discharge min(s, pbar) at price 10).  Interpolating V_1 at s0 = 0.3 (x = 0.6) gives
    0.4*0 + 0.6*5 = 3 = lambda*s0; s0 = 0.8 (x = 1.6) gives 0.4*5 + 0.6*10 = 8 = lambda*s0.  A
    swapped weight (w vs 1 - w) gives 2 and 7 instead."""
    pr = simple_problem(1.0, 2.0, 0.5, 1.0, T=1, lam=[10.0], s0=s0)
    sol = _solve(pr)
    assert sol.V[0, 0].tolist() == [0.0, 5.0, 10.0, 10.0, 10.0]
    assert abs(sol.J - J_closed) <= 1e-12
    assert abs(oracle.objective(pr, sol.V[0]) - J_closed) <= 1e-12


@pytest.mark.parametrize("seed", range(16))
def test_objective_off_grid_s0_exact_expectimax(seed):
    """V7 at an off-grid s0: the exact-rational expectimax with a start lottery between the two
    neighbouring grid states equals the oracle's interpolated J."""
    inst = workloads.random_instance(seed, T=None, K=None, S_max=8)
    rng = np.random.Generator(np.random.PCG64(seed + 99))
    x = float(rng.integers(0, inst.S - 1)) + float(rng.choice([0.125, 0.25, 0.375, 0.7, 0.9]))
    inst = dataclasses.replace(inst, s0=x * inst.delta)
    pr = to_oracle(inst)
    act = oracle.actions(pr)
    sol = _solve(pr)
    J_exact, _ = pins.expectimax_exact(inst, act)
    assert abs(sol.J - float(J_exact)) <= 1e-12 * max(1.0, abs(float(J_exact))), seed
