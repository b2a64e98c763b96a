"""Pins of the oracle's grid and transition tables (Alg. 1 lines 1-5, Eq. 10)."""
import math
import os

import numpy as np
import pytest

import oracle
import pins
import workloads
from helpers import to_oracle, simple_problem

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _rows(name):
    with open(os.path.join(GOLD, name)) as f:
        return [l.split() for l in f if l.strip() and not l.startswith("#")]


def test_table1_action_counts():
    """Table 1: P = 22/42/103/203 at delta = 0.10/0.05/0.02/0.01."""
    eta = math.sqrt(0.85)
    for d, Pn in _rows("table1_actions.txt"):
        pr = simple_problem(pbar=1.0, sbar=4.0, delta=float(d), eta=eta)
        S, A = oracle.dims(pr)
        assert A == int(Pn)


def test_table3_sizes():
    """Table 3: every (S, P) pair, 4/20/100-hour durations at pbar = 1."""
    eta = math.sqrt(0.85)
    for dur, d, S_, P_ in _rows("table3_sizes.txt"):
        pr = simple_problem(pbar=1.0, sbar=float(dur), delta=float(d), eta=eta)
        S, A = oracle.dims(pr)
        assert (S, A) == (int(S_), int(P_))


def test_spec_grid_examples():
    """S:113-124 worked examples."""
    pr = simple_problem(pbar=1.0, sbar=1.0, delta=0.5, eta=1.0)
    assert oracle.actions(pr).tolist() == [-1.0, -0.5, 0.0, 0.5, 1.0]
    pr = simple_problem(pbar=1.0, sbar=1.0, delta=0.5, eta=0.5)
    assert oracle.actions(pr).tolist() == [-1.0, 0.0, 0.25, 0.5, 0.75, 1.0]
    assert oracle.dims(simple_problem(pbar=1.0, sbar=4.0, delta=0.1, eta=1.0))[0] == 41
    assert oracle.status_of(simple_problem(pbar=1.0, sbar=1.0, delta=0.3, eta=1.0)) == oracle.REF_E_CONFIG


@pytest.mark.parametrize("pbar,eta_c,eta_d,delta", [
    (1.0, math.sqrt(0.85), math.sqrt(0.85), 0.1), (99.0, 0.95, 0.95, 1.0), (199.0, 0.95, 0.95, 1.0),
    (9.5, math.sqrt(0.85), math.sqrt(0.85), 1.0), (10.0, 1.0, 1.0, 1.0), (1.0, 0.9, 0.8, 0.25)])
def test_actions_match_independent_eq10(pbar, eta_c, eta_d, delta):
    """The oracle's Eq. 10 equals an independent numpy transcription bit for bit."""
    pr = simple_problem(pbar=pbar, sbar=4 * pbar, delta=delta, eta=eta_c, eta_d=eta_d)
    ref = pins.paper_actions(pbar, eta_c, eta_d, delta)
    got = oracle.actions(pr)
    assert np.array_equal(got, ref)
    assert got[0] == -pbar and got[-1] == pbar and np.all(np.diff(got) > 0)


def test_cfg2_recombination_and_endpoints():
    """interior columns recombine exactly (weight 0); only +-pbar interpolate.
    cfg2 (pbar/delta=99, eta=0.95): A=201, e_c = +94.05, e_d = -104.2105..."""
    inst = workloads.cfg2(T=2, K=2)
    pr = to_oracle(inst)
    S, A = oracle.dims(pr)
    assert (S, A) == (1001, 201)
    tb = oracle.tables(pr)
    assert np.all(tb["w"][1:-1] == 0.0)
    assert tb["off"][0] == 94 and abs(tb["w"][0] - 0.05) < 1e-12
    assert tb["off"][-1] == -105 and abs(tb["w"][-1] - (1 - 99 / 0.95 + 104)) < 1e-12
    # interior offsets are consecutive integers +94 ... -104 (a = 1 .. A-2)
    assert np.array_equal(tb["off"][1:-1], np.arange(94, -105, -1))
    assert np.array_equal(tb["omw"], 1.0 - tb["w"])


def test_spec_mask_examples():
    """grid (sbar=1, delta=0.5, pbar=1, eta=1): infeasible masks of rows s=0 and s=1."""
    pr = simple_problem(pbar=1.0, sbar=1.0, delta=0.5, eta=1.0)
    tb = oracle.tables(pr)
    feas = lambda i: [bool(tb["ilo"][a] <= i <= tb["ihi"][a]) for a in range(5)]
    assert [not f for f in feas(0)] == [False, False, False, True, True]
    assert [not f for f in feas(2)] == [True, True, False, False, False]


@pytest.mark.parametrize("seed", range(40))
def test_mask_agrees_with_eq4_interval(seed):
    """Feasible rows == {i : p_a in P(s_i)} with P(s) the closed-form interval of Eq. 4."""
    inst = workloads.random_instance(seed, S_max=30)
    pr = to_oracle(inst)
    S, A = oracle.dims(pr)
    act = oracle.actions(pr)
    tb = oracle.tables(pr)
    for i in range(S):
        s = i * inst.delta
        lo = -min(inst.pbar, (inst.sbar - s) / inst.eta_c)
        hi = min(inst.pbar, s * inst.eta_d)
        for a in range(A):
            in_int = lo - 1e-9 * inst.delta <= act[a] <= hi + 1e-9 * inst.delta
            feas = tb["ilo"][a] <= i <= tb["ihi"][a]
            assert in_int == feas, (seed, i, a)


def test_validation_errors():
    base = dict(pbar=1.0, sbar=4.0, delta=0.1, eta=1.0)
    assert oracle.status_of(simple_problem(**base)) == 0
    for bad in [dict(eta=0.0), dict(eta=1.5), dict(sbar=4.05), dict(delta=-1.0), dict(pbar=0.0)]:
        kw = dict(base); kw.update(bad)
        assert oracle.status_of(simple_problem(**kw)) == oracle.REF_E_CONFIG, bad
    pr = simple_problem(**base)
    pr.lam = np.array([[np.nan]])
    assert oracle.status_of(pr) == oracle.REF_E_DATA
    pr = simple_problem(**base)
    pr.actions = np.array([-1.0, 0.5, 0.25])          # not ascending
    assert oracle.status_of(pr) == oracle.REF_E_CONFIG
    pr.actions = np.array([-1.0, -0.5, 0.5])          # no zero action
    assert oracle.status_of(pr) == oracle.REF_E_CONFIG
    pr = simple_problem(**base, K=2, T=2)
    pr.P = np.array([[[0.5, 0.6], [0.5, 0.5]]])       # row not a simplex
    assert oracle.status_of(pr) == oracle.REF_E_DATA


def test_cfg5_shards_cover_the_sweep_once():
    """bench.py --config cfg5 (instance sharding, no data-path collective): with world x n = 1024
    the stratified rank samples cover the 1024-configuration sweep exactly once, and a single rank's sample
    spreads over the whole pbar/eta range (not its cheapest corner)."""
    import workloads
    for world in (1, 2, 4, 8):
        n = 1024 // world
        got = sorted(i for r in range(world) for i in workloads.cfg5_shard(r, world, n))
        assert got == list(range(1024)), world
    idx = workloads.cfg5_shard(0, 1, 128)
    assert idx[0] == 0 and idx[-1] >= 1016 and len(set(idx)) == 128
    sweep = workloads.cfg5_sweep()
    ratios = [sweep[i]["pbar"] for i in idx]
    assert min(ratios) < 11.0 and max(ratios) > 95.0
