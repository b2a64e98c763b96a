"""Independent reference computations used to PIN the oracle (tests only).

Nothing here calls oracle/ or the product: each function is a separate formulation of what
the paper defines, so that a mistake in the oracle (a dropped term, a wrong sign or index,
a transposed operand) shows up as a disagreement:

* ``paper_actions``       -- Eq. 10 in numpy, for the grid pins.
* ``alg1_numpy``          -- a literal transliteration of Algorithm 1 with the
                             garble readings R1-R4; the stagewise-independent (rank-1) case.
* ``expectimax_exact``    -- top-down Bellman recursion (Eqs. 5-6) in exact rational
                             arithmetic (fractions.Fraction), with the grid-MDP lottery at
                             off-grid endpoints (R16).
* ``enumerate_sequences`` -- brute force over all A^T action sequences (K = 1, on-lattice).
* ``lp_value`` / ``milp_value`` -- the deterministic LP of Eq. 1 and the MILP of Eq. 3
                             solved with scipy's HiGHS.
* ``hull_exhaustive``     -- O(n^3) upper-hull vertex test (a point is a vertex iff no chord of
                             two other points lies on or above it).
"""
from __future__ import annotations

import itertools
import math
from fractions import Fraction
from functools import lru_cache

import numpy as np

TOL = 1e-9


def transition(p, eta_c, eta_d):
    """Eq. 2: signed SoC change for net power p (p > 0 discharges)."""
    return -p / eta_d if p >= 0 else -eta_c * p


def paper_actions(pbar, eta_c, eta_d, delta):
    """Eq. 10 with the endpoint clamp (R6)."""
    nc = math.ceil(pbar * eta_c / delta - 1e-9)
    nd = math.ceil(pbar / (delta * eta_d) - 1e-9)
    ch = [-min(j * delta / eta_c, pbar) for j in range(nc, 0, -1)]
    di = [min(j * delta * eta_d, pbar) for j in range(1, nd + 1)]
    return np.array(ch + [0.0] + di)


def alg1_numpy(inst, actions):
    """Algorithm 1, line by line, for stagewise-independent prices.

    Returns the list [V_hat_0, ..., V_hat_{T-1}] of expected value vectors (V_hat_T = 0).
    The paper's R price samples are the K columns of inst.lam; pi_hat_t = inst.pi[t-1]."""
    T, S = inst.T, inst.S
    s_hat = inst.delta * np.arange(S)
    p_hat = np.asarray(actions, dtype=np.float64)
    Fp = np.array([transition(p, inst.eta_c, inst.eta_d) for p in p_hat])
    sigma = s_hat[:, None] + Fp[None, :]                                   # line 2
    z = np.clip(sigma, 0.0, inst.sbar) / inst.delta                       # line 3 (R1, 0-based)
    zm, zp = np.floor(z).astype(np.int64), np.ceil(z).astype(np.int64)    # line 4
    with np.errstate(invalid="ignore", divide="ignore"):
        b = np.where(zp == zm, 0.0, (z - zm) / (zp - zm))                 # line 5 (R4)
    infeasible = (sigma < -TOL * inst.delta) | (sigma > inst.sbar + TOL * inst.delta)
    V_hat = np.zeros(S)                                                   # line 1
    out = [None] * T
    for t in range(T, 0, -1):                                             # R3: t = T..1
        lam_t, pi_t = inst.lam[t - 1], inst.pi[t - 1]
        V_next = (1.0 - b) * V_hat[zm] + b * V_hat[zp]                    # line 7
        V_next[infeasible] = -np.inf                                      # line 8 (R2)
        Q_all = p_hat[None, :, None] * lam_t[None, None, :] + V_next[:, :, None]   # line 9
        Q = Q_all.max(axis=1)                                             # line 10
        V_hat = Q @ pi_t                                                  # line 11
        out[t - 1] = V_hat
    return out


def _frac(x):
    return Fraction(x) if not isinstance(x, Fraction) else x


def expectimax_exact(inst, actions, i0=None, payoff=None):
    """Top-down expectimax over (t, i, k) in exact rational arithmetic.

    Next state of action p at grid state i: z = i + F(p)/delta (exact); if z is within 1e-9 of an
    integer it is that integer (R6/R7), otherwise a lottery between floor(z) and floor(z)+1 with
    weight z - floor(z) (R16).  payoff(t, k, a) -> Fraction overrides lambda p (default)."""
    T, K, S = inst.T, inst.K, inst.S
    delta = _frac(inst.delta)
    acts = [_frac(a) for a in actions]
    eta_c, eta_d = _frac(inst.eta_c), _frac(inst.eta_d)
    lam = [[_frac(x) for x in row] for row in np.asarray(inst.lam)]

    def trans(p):
        return -p / eta_d if p >= 0 else -eta_c * p

    moves = []
    for p in acts:
        e = trans(p) / delta
        r = round(e)
        if abs(e - r) <= Fraction(1, 10**9):
            moves.append((int(r), Fraction(0)))
        else:
            f = math.floor(e)
            moves.append((f, e - f))
    if inst.P is None:
        Pm = None
        pis = [[_frac(x) for x in row] for row in np.asarray(inst.pi)]
    else:
        Pm = [[[_frac(x) for x in row] for row in mat] for mat in np.asarray(inst.P)]
        pis = [_frac(x) for x in np.asarray(inst.pi)]

    def pay(t, k, a):
        if payoff is not None:
            return payoff(t, k, a)
        return lam[t - 1][k] * acts[a]

    @lru_cache(maxsize=None)
    def Vk(t, i, k):            # value after observing k at stage t, state i
        best = None
        for a, (o, w) in enumerate(moves):
            lo, hi = i + o, i + o + (1 if w else 0)
            if lo < 0 or hi > S - 1:
                continue
            cont = (1 - w) * EV(t, lo, k) + (w * EV(t, hi, k) if w else 0)
            c = pay(t, k, a) + cont
            if best is None or c > best:
                best = c
        return best

    @lru_cache(maxsize=None)
    def EV(t, i, k):            # expected value of V_{t+1}(i, .) given k_t = k
        if t == T:
            return Fraction(0)
        if Pm is None:
            row = pis[t]
        else:
            row = Pm[t - 1][k]
        return sum((row[kp] * Vk(t + 1, i, kp) for kp in range(K)), Fraction(0))

    pi1 = pis[0] if Pm is None else pis
    if i0 is None:
        # R24: an off-grid s0 is a start lottery between the two neighbouring grid
        # states, floor(x) w.p. 1 - w and floor(x) + 1 w.p. w, w = x - floor(x) (exact rationals).
        x = _frac(inst.s0) / delta
        r = round(x)
        if abs(x - r) <= Fraction(1, 10**9):
            starts = [(int(r), Fraction(1))]
        else:
            f = math.floor(x)
            starts = [(f, 1 - (x - f)), (f + 1, x - f)]
    else:
        starts = [(i0, Fraction(1))]
    J = sum((pi1[k] * q * Vk(1, i, k) for k in range(K) for i, q in starts), Fraction(0))
    expectimax_exact.last = dict(EV=EV, moves=moves, pay=pay)
    return J, Vk


def enumerate_sequences(prices, actions, sbar, s0, eta_c, eta_d, tol=1e-9):
    """Max of sum_t lambda_t p_t over ALL action sequences whose continuous SoC path stays in
    [0, sbar] (Eqs. 1-2); exact discretized optimum when no interpolation occurs."""
    best = -math.inf
    for seq in itertools.product(range(len(actions)), repeat=len(prices)):
        s, val, ok = s0, 0.0, True
        for lam, a in zip(prices, seq):
            p = actions[a]
            s = s + transition(p, eta_c, eta_d)
            if s < -tol or s > sbar + tol:
                ok = False
                break
            val += lam * p
        if ok and val > best:
            best = val
    return best


def lp_value(prices, pbar, sbar, s0, eta_c, eta_d, restrict_neg=False, integer=False):
    """max sum lambda_t (p^d_t - p^c_t) s.t. Eq. 1 bounds and Eq. 3's SoC recursion with
    separate p^c, p^d.  integer=True adds the binary z_t of Eq. 3 (MILP);
    restrict_neg=True fixes p^d_t = 0 where lambda_t <= 0 (the LP restriction)."""
    from scipy.optimize import Bounds, LinearConstraint, milp
    T = len(prices)
    # variables: pc[0..T), pd[0..T), s[0..T), z[0..T) (z only if integer)
    nz = T if integer else 0
    n = 3 * T + nz
    c = np.zeros(n)
    c[:T] = np.asarray(prices)          # minimize -(sum lam (pd - pc)) = sum lam pc - lam pd
    c[T:2 * T] = -np.asarray(prices)
    lb = np.zeros(n)
    ub = np.concatenate([np.full(T, pbar), np.full(T, pbar), np.full(T, sbar), np.ones(nz)])
    if restrict_neg:
        for t in range(T):
            if prices[t] <= 0:
                ub[T + t] = 0.0
    rows, lo, hi = [], [], []
    for t in range(T):                  # s_t - s_{t-1} - eta_c pc_t + pd_t / eta_d = 0
        r = np.zeros(n)
        r[2 * T + t] = 1.0
        if t > 0:
            r[2 * T + t - 1] = -1.0
        r[t] = -eta_c
        r[T + t] = 1.0 / eta_d
        rows.append(r)
        v = s0 if t == 0 else 0.0
        lo.append(v); hi.append(v)
    if integer:
        for t in range(T):              # pc <= pbar z ; pd <= pbar (1 - z)
            r = np.zeros(n); r[t] = 1.0; r[3 * T + t] = -pbar
            rows.append(r); lo.append(-np.inf); hi.append(0.0)
            r = np.zeros(n); r[T + t] = 1.0; r[3 * T + t] = pbar
            rows.append(r); lo.append(-np.inf); hi.append(pbar)
    integrality = np.concatenate([np.zeros(3 * T), np.ones(nz)])
    res = milp(c, constraints=LinearConstraint(np.array(rows), lo, hi), bounds=Bounds(lb, ub),
               integrality=integrality, options=dict(mip_rel_gap=1e-12))
    assert res.success, res.message
    pc, pd = res.x[:T], res.x[T:2 * T]
    compl = int(np.sum((pc > 1e-7) & (pd > 1e-7)))
    return -res.fun, compl


def hull_exhaustive(ps, us):
    """Indices of upper-hull vertices of points with strictly increasing ps, O(n^3):
    j is a vertex iff j is an endpoint, or no chord (l, r) with l < j < r lies on or above it.
    Exact rational arithmetic so collinear points are decided exactly."""
    P = [Fraction(x) for x in ps]
    U = [Fraction(x) for x in us]
    n = len(P)
    out = []
    for j in range(n):
        if j in (0, n - 1):
            out.append(j)
            continue
        dominated = False
        for l in range(j):
            for r in range(j + 1, n):
                chord = U[l] + (U[r] - U[l]) * (P[j] - P[l]) / (P[r] - P[l])
                if chord >= U[j]:
                    dominated = True
                    break
            if dominated:
                break
        if not dominated:
            out.append(j)
    return out
