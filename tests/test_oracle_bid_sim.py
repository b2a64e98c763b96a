"""Pins of the oracle's bid curves (Eqs. 7-12) and forward simulation."""
import os

import numpy as np
import pytest

import oracle
import pins
import workloads
from helpers import to_oracle, simple_problem

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _W_problem(W_row, sbar, delta):
    """A T=1, K=1 problem plus a hand-made W_1 row, to exercise the hull on chosen points."""
    pr = simple_problem(1.0, sbar, delta, 1.0, T=1, K=1, lam=[0.0])
    W = np.asarray(W_row, dtype=np.float64).reshape(1, 1, -1)
    return pr, W


def test_spec_bid_examples():
    """S:315 (points), S:323 (dent removed), S:331 (prices), S:342 (clearing)."""
    # bid1: V row [0, 1, 4], s = 0.5 on (sbar=1, delta=0.5): points (-0.5, 4), (0, 1), (0.5, 0)
    pr, W = _W_problem([0.0, 1.0, 4.0], 1.0, 0.5)
    c = oracle.bidcurve(pr, W, 1, 1, 0)
    assert c["q"].tolist() == [-0.5, 0.0, 0.5] or c["q"].tolist() == [-0.5, 0.5]
    # the three points are not concave in p (slopes -6, -2): middle point is a dent -> removed
    assert c["q"].tolist() == [-0.5, 0.5] and c["price"].tolist() == [4.0]   # -(0 - 4)/(0.5 + 0.5)
    # bid2: (0,0), (1,-2), (2,0) scaled onto the grid: u = (0, -2, 0) at p = (-0.5, 0, 0.5)
    pr, W = _W_problem([0.0, -2.0, 0.0], 1.0, 0.5)
    c = oracle.bidcurve(pr, W, 1, 1, 0)
    assert c["q"].tolist() == [-0.5, 0.5] and c["price"].tolist() == [0.0]
    # bid3: hull (-1, 9), (0, 5), (1, 0) -> prices [4, 5]; (sbar=2, delta=1), i = 1
    pr, W = _W_problem([0.0, 5.0, 9.0], 2.0, 1.0)
    c = oracle.bidcurve(pr, W, 1, 1, 0)
    assert c["q"].tolist() == [-1.0, 0.0, 1.0] and c["price"].tolist() == [4.0, 5.0]
    # bid4: clearing at 4.5 -> quantity 0; ties (lambda == 4) go to the larger quantity (R9)
    assert c["q"][oracle.clear(c, 4.5)] == 0.0
    assert c["q"][oracle.clear(c, 4.0)] == 0.0
    assert c["q"][oracle.clear(c, 3.99)] == -1.0
    assert c["q"][oracle.clear(c, 5.0)] == 1.0


@pytest.mark.parametrize("seed", range(25))
def test_hull_matches_exhaustive(seed):
    """the monotone-chain hull equals an O(n^3) exhaustive vertex test on random profiles."""
    rng = np.random.default_rng(seed)
    n = 11
    row = np.round(rng.normal(0, 5, size=n), 1) if seed % 2 else rng.normal(0, 5, size=n)
    pr, W = _W_problem(row, 10.0, 1.0)
    act = oracle.actions(pr)
    i = int(rng.integers(0, n))
    c = oracle.bidcurve(pr, W, 1, i, 0)
    tb = oracle.tables(pr)
    feas = [a for a in range(len(act)) if tb["ilo"][a] <= i <= tb["ihi"][a]]
    ps = [act[a] for a in feas]
    us = [row[i + tb["off"][a]] for a in feas]
    ref = [feas[j] for j in pins.hull_exhaustive(ps, us)]
    assert c["vert"].tolist() == ref
    assert np.all(np.diff(c["price"]) >= 0)


@pytest.mark.parametrize("seed", range(10))
def test_bid_curve_consistent_with_stencil(seed):
    """V15: with lambda p - g(p) payoffs, max over hull vertices of (lambda p + u) equals V_t(i, k)
    (to rounding), the clearing quantity attains it, and clearing is monotone in the price."""
    inst = workloads.random_instance(seed + 300, S_max=25, T=4, K=3)
    pr = to_oracle(inst)
    S, A = oracle.dims(pr)
    if seed % 2:
        inst.payoff_kind, inst.g = workloads.PAYOFF_LINEAR_MINUS_G, workloads.random_g(seed, A, 30.0)
        pr = to_oracle(inst)
    sol = oracle.backward(pr)
    for t in range(1, inst.T + 1):
        for k in range(inst.K):
            lam = inst.lam[t - 1, k]
            for i in range(S):
                c = oracle.bidcurve(pr, sol.W, t, i, k)
                vals = [lam * q + u for q, u in zip(c["q"], _hull_u(pr, sol.W, t, i, k, c))]
                v = sol.V[t - 1, k, i]
                assert abs(max(vals) - v) <= 1e-9 * max(1.0, abs(v))
                j = oracle.clear(c, lam)
                assert abs(vals[j] - v) <= 1e-9 * max(1.0, abs(v))
                assert np.all(np.diff(c["price"]) >= 0)
                qs = [c["q"][oracle.clear(c, x)] for x in np.linspace(-200, 200, 41)]
                assert np.all(np.diff(qs) >= 0)


def _hull_u(pr, W, t, i, k, c):
    tb = oracle.tables(pr)
    Wrow = W[t - 1, k]
    g = pr.g if pr.payoff_kind == workloads.PAYOFF_LINEAR_MINUS_G else None
    out = []
    for a in c["vert"]:
        o, w = tb["off"][a], tb["w"][a]
        u = Wrow[i + o] if w == 0 else tb["omw"][a] * Wrow[i + o] + w * Wrow[i + o + 1]
        out.append(u - (g[a] if g is not None else 0.0))
    return out


def test_terminal_stage_prices_zero():
    """terminal-stage curve (W_T = 0, linear payoff) has all segment prices 0."""
    inst = workloads.cfg1("b")
    pr = to_oracle(inst)
    sol = oracle.backward(pr)
    for i in [0, 10, 50, 100]:
        c = oracle.bidcurve(pr, sol.W, inst.T, i, 2)
        assert np.all(c["price"] == 0.0)


def test_philox_known_answers():
    """V17: Random123 known-answer vectors (tests/golden/philox_kat.txt)."""
    with open(os.path.join(GOLD, "philox_kat.txt")) as f:
        rows = [l.split() for l in f if l.strip() and not l.startswith("#")]
    for r in rows:
        v = [int(x, 16) for x in r]
        assert oracle.philox(v[0:4], v[4:6]) == v[6:10]


@pytest.mark.parametrize("name", ["cfg1a", "cfg1b", "cfg1b-rank1"])
def test_simulation_mean_matches_J(name):
    """V16: under lottery semantics E[profit] = J exactly, so the Monte Carlo mean lies within
    5 standard errors of J."""
    inst = workloads.cfg1(name[4], rank1=name.endswith("rank1"))
    pr = to_oracle(inst)
    sol = oracle.backward(pr)
    n = 20000
    per, m, v = oracle.simulate(pr, sol.pol, n, seed=12345)
    se = np.sqrt(v / n)
    assert abs(m - sol.J) <= 5 * se + 1e-9
    assert m == np.sum(per) / n or abs(m - np.mean(per)) < 1e-9 * abs(m)


def test_simulation_deterministic_path_equals_J():
    """K = 1, on-lattice: every path is the same deterministic optimal schedule, profit == J."""
    inst = workloads.random_instance(42, T=8, K=1, S_max=20, lattice=True, rank1=False)
    pr = to_oracle(inst)
    sol = oracle.backward(pr)
    per, m, v = oracle.simulate(pr, sol.pol, 16, seed=1)
    assert np.all(np.abs(per - sol.J) <= 1e-9 * max(1.0, abs(sol.J)))
    assert v <= 1e-18 * max(1.0, sol.J ** 2)


# ---- simulation modes (SURVEY §8(a) a7 "(or clear the bid)", §8(c) step 7 physical mode; R25/R26) ----

@pytest.mark.parametrize("seed", range(6))
def test_physical_mode_equals_lottery_on_the_lattice(seed):
    """V21: with eta = 1 and integral pbar/delta every action lands on the grid, so re-optimising at
    the real SoC is the policy lookup: the physical and lottery paths agree to the bit."""
    inst = workloads.random_instance(300 + seed, T=6, K=1 + seed % 3, S_max=30, lattice=True)
    pr = to_oracle(inst)
    sol = oracle.backward(pr)
    lot, _, _ = oracle.simulate(pr, sol.pol, 500, seed=9)
    phy, _, _ = oracle.simulate_mode(pr, sol.pol, sol.W, oracle.SIM_PHYSICAL, 500, seed=9)
    assert np.array_equal(lot, phy)


def test_physical_mode_single_stage_closed_form():
    """T = 1 (W_1 = 0): the physical decision at s0 = sbar is the largest feasible discharge,
    min(pbar, sbar eta_d) (Eq. 1 and Eq. 4 on the real state); profit lambda times it."""
    for eta, s0 in ((0.9, 3.0), (0.8, 1.0), (1.0, 2.0)):
        inst = workloads.random_instance(5, T=1, K=1, S_max=6)
        inst.eta_c = inst.eta_d = eta
        inst.delta, inst.sbar, inst.s0, inst.pbar = 1.0, 5.0, s0, 2.0
        inst.lam = np.array([[7.0]])
        inst.pi = np.array([1.0])
        inst.P = None if inst.P is None else np.zeros((0, 1, 1))
        pr = to_oracle(inst)
        sol = oracle.backward(pr)
        act = oracle.actions(pr)
        feas = [p for p in act if 0 <= s0 - (p / eta if p >= 0 else eta * p) <= 5.0]
        per, _, _ = oracle.simulate_mode(pr, sol.pol, sol.W, oracle.SIM_PHYSICAL, 3, seed=1)
        assert np.all(per == 7.0 * max(feas)), (per, feas)
        assert max(feas) == pytest.approx(min(2.0, s0 * eta) if s0 * eta < 2.0 else max(a for a in act if a <= 2.0))


def test_physical_mode_below_lp_bound():
    """K = 1 deterministic prices, eta < 1: the physical schedule is a feasible continuous schedule,
    so its profit never exceeds the LP optimum (scipy HiGHS)."""
    from pins import lp_value
    inst = workloads.random_instance(77, T=8, K=1, S_max=25, rank1=False)
    inst.eta_c = inst.eta_d = 0.9
    pr = to_oracle(inst)
    sol = oracle.backward(pr)
    per, _, _ = oracle.simulate_mode(pr, sol.pol, sol.W, oracle.SIM_PHYSICAL, 4, seed=3)
    lp, _ = lp_value(inst.lam[:, 0], inst.pbar, inst.sbar, inst.s0, 0.9, 0.9)
    assert np.all(per <= lp + 1e-9 * max(1.0, abs(lp)))
    assert np.all(per == per[0])          # deterministic prices: every path the same


@pytest.mark.parametrize("name", ["cfg1b", "cfg1b-rank1"])
def test_clear_bids_mode_follows_the_policy(name):
    """Clearing the stage's bid curve at the realised price selects the hull vertex that maximises
    lambda p + u (Eq. 12 / merit order) -- the argmax policy except on exact ties:
    (almost) every path equals the lottery path, and the mean lies within 5 standard errors of J."""
    inst = workloads.cfg1("b", rank1=name.endswith("rank1"))
    pr = to_oracle(inst)
    sol = oracle.backward(pr)
    n = 4000
    lot, _, _ = oracle.simulate(pr, sol.pol, n, seed=21)
    clr, m, v = oracle.simulate_mode(pr, sol.pol, sol.W, oracle.SIM_CLEAR_BIDS, n, seed=21)
    assert np.mean(lot == clr) >= 0.99
    assert abs(m - sol.J) <= 5 * np.sqrt(v / n) + 1e-9


def test_clear_bids_mode_rejects_table_payoffs():
    inst = workloads.random_instance(8, T=3, K=2, S_max=8)
    pr0 = to_oracle(inst)
    S, A = oracle.dims(pr0)
    inst.payoff_kind = workloads.PAYOFF_TABLE
    inst.g = workloads.random_table(8, inst.T, inst.K, A)
    pr = to_oracle(inst)
    sol = oracle.backward(pr)
    with pytest.raises(oracle.OracleError):
        oracle.simulate_mode(pr, sol.pol, sol.W, oracle.SIM_CLEAR_BIDS, 4, seed=1)


# ---- dispatch strategies of the Fig. 3 study (NEXT-2; R27/R28) ----

def _det_instance(lam, seed=3):
    inst = workloads.random_instance(seed, T=len(lam), K=1, S_max=40)
    inst.eta_c = inst.eta_d = 0.9
    inst.lam = np.asarray(lam, float).reshape(-1, 1)
    inst.pi = np.ones((len(lam), 1)) if inst.P is None else np.array([1.0])
    if inst.P is not None:
        inst.P = np.ones((len(lam) - 1, 1, 1))
    return inst


def test_strategy_physical_equals_physical_mode():
    inst = workloads.cfg1("b")
    pr = to_oracle(inst)
    sol = oracle.backward(pr)
    a, _ = oracle.simulate_strategy(pr, sol.W, oracle.SIM_PHYSICAL, 300, seed=8)
    b, _, _ = oracle.simulate_mode(pr, sol.pol, sol.W, oracle.SIM_PHYSICAL, 300, seed=8)
    assert np.array_equal(a, b)


def test_self_scheduled_equals_bids_when_the_lag_is_exact():
    """R27: with prices constant over time the lagged price is the realised one, so the self-scheduled
    decisions are the re-optimised ones (SPEC: 'lagged == realized -> identical to simulateBidding')."""
    inst = _det_instance([7.5] * 9)
    pr = to_oracle(inst)
    sol = oracle.backward(pr)
    a, _ = oracle.simulate_strategy(pr, sol.W, oracle.SIM_PHYSICAL, 5, seed=2)
    b, _ = oracle.simulate_strategy(pr, sol.W, oracle.SIM_SELF, 5, seed=2)
    assert np.array_equal(a, b)


def test_self_scheduled_loses_on_anticorrelated_lags():
    """Alternating prices make the lagged price the wrong forecast: self-scheduling earns less than
    re-optimising at the realised price (Fig. 3 ordering 'DP bid curves > self-scheduled')."""
    inst = _det_instance([1.0, 40.0] * 6)
    pr = to_oracle(inst)
    sol = oracle.backward(pr)
    a, _ = oracle.simulate_strategy(pr, sol.W, oracle.SIM_PHYSICAL, 3, seed=2)
    b, _ = oracle.simulate_strategy(pr, sol.W, oracle.SIM_SELF, 3, seed=2)
    assert np.all(b < a)


def test_fixed_schedule_replays_and_settles_linearly():
    """R28: the physical plan of a deterministic problem, replayed as a fixed schedule, earns the same;
    settled at doubled prices (g = 0) it earns exactly twice (SPEC: linear settlement)."""
    lam = [12.0, 3.0, 25.0, 9.0, 31.0, 2.0, 18.0]
    inst = _det_instance(lam)
    pr = to_oracle(inst)
    sol = oracle.backward(pr)
    phy, act = oracle.simulate_strategy(pr, sol.W, oracle.SIM_PHYSICAL, 1, seed=4, want_actions=True)
    fix, _ = oracle.simulate_strategy(pr, None, oracle.SIM_FIXED, 1, seed=4, schedule=act[:, 0])
    assert np.array_equal(phy, fix)
    inst2 = _det_instance([2 * x for x in lam])
    fix2, _ = oracle.simulate_strategy(to_oracle(inst2), None, oracle.SIM_FIXED, 1, seed=4, schedule=act[:, 0])
    assert fix2[0] == 2 * fix[0]


@pytest.mark.parametrize("s0, J_closed", [(0.3, 3.0), (0.8, 8.0)])
def test_simulation_off_grid_start_lottery(s0, J_closed):
    """R24 in the simulation: an off-grid s0 starts at floor(x) w.p. 1 - w and floor(x) + 1 w.p. w,
    so the Monte Carlo mean is the closed-form J = lambda*s0 (T = 1, lambda = 10, V_1 = [0, 5, 10,
    10, 10]; see test_objective_off_grid_s0_closed_form).  A swapped start weight would move the
    mean by 1.0, about 40 standard errors at n = 20000."""
    pr = simple_problem(1.0, 2.0, 0.5, 1.0, T=1, lam=[10.0], s0=s0)
    sol = oracle.backward(pr)
    n = 20000
    per, m, v = oracle.simulate(pr, sol.pol, n, seed=777)
    se = np.sqrt(v / n)
    assert 0.0 < se < 0.05
    assert abs(m - J_closed) <= 5 * se
    assert set(np.unique(per).tolist()) <= {0.0, 5.0, 10.0}


def test_simulation_off_grid_start_multistage():
    """R24 with a multi-stage Markov instance: the MC mean from an off-grid s0 lies within 5 standard
    errors of the exact-rational expectimax J (start lottery), not only of the oracle's own J."""
    import dataclasses
    inst = workloads.random_instance(5, T=4, K=2, S_max=10, rank1=False)
    inst = dataclasses.replace(inst, s0=(min(3, inst.S - 2) + 0.375) * inst.delta)
    pr = to_oracle(inst)
    sol = oracle.backward(pr)
    J_exact, _ = pins.expectimax_exact(inst, oracle.actions(pr))
    n = 40000
    per, m, v = oracle.simulate(pr, sol.pol, n, seed=4242)
    se = np.sqrt(v / n)
    assert abs(m - float(J_exact)) <= 5 * se + 1e-9
