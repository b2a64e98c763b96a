"""Seeded synthetic inputs shared by the oracle tests and the CUDA path.

This module holds NO arithmetic of the method (no grid, no transition table, no DP step):
it only draws the problem data of the paper's workloads -- price levels lambda_{t,k},
transition matrices P_t, initial distributions, payoff tables -- with the shapes and value
distributions of DESIGN.md §4 (the "ISO-NE-shaped" recipe of SURVEY.md §8(d).1).  The action
grid (Eq. 10) is computed independently inside each implementation from (pbar, eta, delta).

Every function is a pure function of its arguments and seed.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from statistics import NormalDist

import numpy as np

PAYOFF_LINEAR, PAYOFF_LINEAR_MINUS_G, PAYOFF_TABLE = 0, 1, 2
SEED_BASE = 2511_15629


@dataclass
class Instance:
    """Everything a solver needs; field names follow esdp_problem (include/esdp.h)."""
    name: str
    T: int
    K: int
    pbar: float
    sbar: float
    s0: float
    eta_c: float
    eta_d: float
    delta: float
    lam: np.ndarray                      # [T][K]
    P: np.ndarray | None                 # [T-1][K][K] row-stochastic, or None (rank-1)
    pi: np.ndarray                       # [K] (Markov) or [T][K] (rank-1 per-stage marginals)
    actions: np.ndarray | None = None    # None => paper grid (Eq. 10)
    payoff_kind: int = PAYOFF_LINEAR
    g: np.ndarray | None = None
    meta: dict = field(default_factory=dict)

    @property
    def S(self) -> int:  # size of the state grid, only for sizing buffers in harnesses
        return int(round(self.sbar / self.delta)) + 1


# ---------------------------------------------------------------------------------------------
# ISO-NE-shaped price chain (the paper's data, is not available)
# ---------------------------------------------------------------------------------------------

def da_shape(h: np.ndarray) -> np.ndarray:
    """Hour-of-day day-ahead shape mu(h) in $/energy unit (morning ramp + evening peak)."""
    return (38.0 + 12.0 * np.sin(2 * np.pi * (h - 9.0) / 24.0)
            + 25.0 * np.exp(-((h - 18.5) / 1.5) ** 2) - 8.0 * np.exp(-((h - 4.0) / 2.0) ** 2))


def _mixture_cdf(x: float) -> float:
    """CDF of 0.9 Laplace(0, 6) + 0.1 Laplace(0, 40) (heavy-tailed RT-DA spread)."""
    def lap(x, b):
        return 0.5 * math.exp(x / b) if x < 0 else 1.0 - 0.5 * math.exp(-x / b)
    return 0.9 * lap(x, 6.0) + 0.1 * lap(x, 40.0)


def spread_quantiles(K: int) -> np.ndarray:
    """q_k = F^{-1}((k + 0.5)/K) of the spread mixture (quantile rule of S:470), by bisection."""
    out = np.empty(K)
    for k in range(K):
        target = (k + 0.5) / K
        lo, hi = -2000.0, 2000.0
        for _ in range(200):
            mid = 0.5 * (lo + hi)
            if _mixture_cdf(mid) < target:
                lo = mid
            else:
                hi = mid
        out[k] = 0.5 * (lo + hi)
    return out


def ar1_transition(K: int, rho: float) -> np.ndarray:
    """Gaussian-copula AR(1) on the quantile index: P[k][k'] ∝ exp(-(z_k' - rho z_k)^2 / (2(1-rho^2)))."""
    nd = NormalDist()
    z = np.array([nd.inv_cdf((k + 0.5) / K) for k in range(K)])
    if K == 1:
        return np.ones((1, 1))
    d = z[None, :] - rho * z[:, None]
    logits = -(d * d) / (2.0 * (1.0 - rho * rho))
    logits -= logits.max(axis=1, keepdims=True)
    M = np.exp(logits)
    M /= M.sum(axis=1, keepdims=True)
    return M


def price_chain(T: int, K: int, stage_hours: float, rho: float | None = None, per_stage_rho: bool = False,
                seed: int = SEED_BASE, jitter: float = 0.01, season: bool = False):
    """lambda[T][K], P[T-1][K][K], pi1[K] for an ISO-NE-shaped Markov price chain."""
    rng = np.random.Generator(np.random.PCG64(seed))
    t = np.arange(T)
    h = (t * stage_hours) % 24.0
    mu = da_shape(h)
    if season:
        day = (t * stage_hours) // 24.0
        mu = mu * (1.0 + 0.25 * np.cos(2 * np.pi * (day - 15.0) / 365.0))
        mu = mu * np.where((day % 7) >= 5, 0.9, 1.0)
    sig = 1.0 + 0.5 * ((h >= 16.0) & (h < 21.0))
    q = spread_quantiles(K)
    lam = mu[:, None] + sig[:, None] * q[None, :]
    if jitter:
        lam = lam * (1.0 + jitter * rng.uniform(-1.0, 1.0, size=lam.shape))
    if rho is None:
        rho = 0.95 if stage_hours < 1.0 else 0.7
    if T > 1:
        if per_stage_rho:
            P = np.stack([ar1_transition(K, 0.7 + 0.2 * math.sin(2 * math.pi * (s + 1) / 24.0))
                          for s in range(T - 1)])
        else:
            P = np.broadcast_to(ar1_transition(K, rho), (T - 1, K, K)).copy()
    else:
        P = np.zeros((0, K, K))
    pi1 = np.full(K, 1.0 / K)
    return np.ascontiguousarray(lam), np.ascontiguousarray(P), pi1


# ---------------------------------------------------------------------------------------------
# BASELINE.json configs
# ---------------------------------------------------------------------------------------------

def cfg1(variant: str = "b", rank1: bool = False) -> Instance:
    """T=24 hourly, S=101, A=21, K=5, linear payoff.  (a): eta=1, pbar/delta=10 (no interpolation);
    (b): eta=sqrt(0.85), pbar/delta=9.5 (endpoints interpolated)."""
    T, K = 24, 5
    lam, P, pi1 = price_chain(T, K, 1.0, seed=SEED_BASE + 1)
    eta, pbar = (1.0, 10.0) if variant == "a" else (math.sqrt(0.85), 9.5)
    if rank1:
        P, pi = None, np.full((T, K), 1.0 / K)
    else:
        pi = pi1
    return Instance(f"cfg1{variant}{'-rank1' if rank1 else ''}", T, K, pbar, 100.0, 0.0, eta, eta, 1.0,
                    lam, P, pi)


def cfg2(s0: float = 500.0, rank1: bool = False, T: int = 288, K: int = 100) -> Instance:
    """ISO-NE-shaped 5-min RT day: T=288, S=1001, A=201, K=100, eta_c=eta_d=0.95 (pbar/delta = 99)."""
    lam, P, pi1 = price_chain(T, K, 5.0 / 60.0, seed=SEED_BASE + 2)
    if rank1:
        P, pi = None, np.full((T, K), 1.0 / K)
    else:
        pi = pi1
    return Instance(f"cfg2{'-rank1' if rank1 else ''}", T, K, 99.0, 1000.0, s0, 0.95, 0.95, 1.0, lam, P, pi)


def cfg3_small() -> Instance:
    """(3i) Table-2 analog: K=1, T=72 hourly, sbar/delta=40, pbar/delta=10,
    eta=sqrt(0.85), s0=sbar, all prices level-shifted <= 0."""
    T = 72
    lam, _, _ = price_chain(T, 1, 1.0, seed=SEED_BASE + 3, jitter=0.0)
    rng = np.random.Generator(np.random.PCG64(SEED_BASE + 30))
    lam = lam + rng.normal(0.0, 8.0, size=lam.shape)
    lam = lam - lam.max()                      # lambda^neg = lambda - max lambda
    eta = math.sqrt(0.85)
    return Instance("cfg3i", T, 1, 10.0, 40.0, 40.0, eta, eta, 1.0, np.ascontiguousarray(lam),
                    np.ones((T - 1, 1, 1)), np.ones(1))


def degradation_g(actions: np.ndarray, c_lin: float = 2.0, c_fix: float = 25.0) -> np.ndarray:
    """g_a = c_lin |p_a| + c_fix [p_a != 0]: linear wear plus a fixed cycling cost (non-concave payoff).
    The caller passes the action vector it will solve on (tests: the oracle's esdp actions, after a
    separate test has pinned the product's action grid to the oracle's bit for bit)."""
    return c_lin * np.abs(actions) + c_fix * (actions != 0.0)


def cfg3_gpu(actions: np.ndarray, T: int = 288, K: int = 100, rank1: bool = False) -> Instance:
    """(3ii) cfg2 dimensions, prices shifted <= 0, non-concave degradation payoff."""
    base = cfg2(T=T, K=K, rank1=rank1)
    lam = base.lam - base.lam.max()
    return Instance(f"cfg3ii{'-rank1' if rank1 else ''}", T, K, base.pbar, base.sbar, base.sbar, 0.95, 0.95,
                    1.0, lam, base.P, base.pi, None, PAYOFF_LINEAR_MINUS_G, degradation_g(actions))


def table1_deterministic(delta: float = 0.01, T: int = 8784, seed: int = SEED_BASE + 6) -> Instance:
    """NEXT-3: Table 1 analog: deterministic prices (K = 1), a 4-hour battery with pbar = 1,
    eta = sqrt(0.85), one year of hourly stages; delta in {0.10, 0.05, 0.02, 0.01} gives
    A = 22 / 42 / 103 / 203 and S = 41 / 81 / 201 / 401 (Table 1 / Table 3 sizes)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    h = np.arange(T) % 24
    day = np.arange(T) // 24
    lam = da_shape(h.astype(np.float64)) * (1.0 + 0.25 * np.cos(2 * np.pi * (day - 15.0) / 365.0))
    lam = lam + rng.laplace(0.0, 6.0, size=T)
    eta = math.sqrt(0.85)
    return Instance(f"table1-delta{delta}", T, 1, 1.0, 4.0, 0.0, eta, eta, delta,
                    np.ascontiguousarray(lam.reshape(T, 1)), np.ones((T - 1, 1, 1)), np.ones(1))


def table3(hours: float = 100.0, delta: float = 0.01, T: int = 8784, R: int = 200,
           seed: int = SEED_BASE + 7) -> Instance:
    """The paper's Table 3 GPU-timing workload with synthetic prices: one year of hourly
    stages, a 1-MW battery of `hours` hours (S = hours/delta + 1; 100 h at delta = 0.01 gives S = 10001,
    A = 203), R = 200 equally likely price samples per hour (stagewise independent: rank-1, pi_t = 1/R,
    S:470), the ISO-NE-shaped hour-of-day/season profile plus spread quantiles."""
    lam, _, _ = price_chain(T, R, 1.0, seed=seed, season=True)
    pi = np.full((T, R), 1.0 / R)
    eta = math.sqrt(0.85)
    return Instance(f"table3-{hours:g}h-delta{delta}", T, R, 1.0, hours, 0.0, eta, eta, delta, lam, None, pi)


def cfg4(T: int = 8760, K: int = 200) -> Instance:
    """Full-year hourly horizon: T=8760, S=2001, A=401, K=200, per-stage P_t (pbar/delta = 199)."""
    lam, P, pi1 = price_chain(T, K, 1.0, per_stage_rho=True, seed=SEED_BASE + 4, season=True)
    return Instance("cfg4", T, K, 199.0, 2000.0, 0.0, 0.95, 0.95, 1.0, lam, P, pi1)


def cfg5_sweep(n: int = 1024):
    """1024 storage configurations: 32 durations x 32 efficiencies on the cfg2 chain."""
    out = []
    ratios = np.geomspace(10.42, 99.0, 32)
    etas = np.linspace(0.80, 0.99, 32)
    for j in range(n):
        out.append(dict(pbar=float(np.round(ratios[j // 32 % 32], 6)), eta=float(etas[j % 32])))
    return out


def cfg5_shard(rank: int, world: int, n: int, total: int = 1024):
    """Sweep indices of rank `rank` of `world` with n configurations per rank: a stratified sample of the
    `total`-configuration sweep (every (world n / total)-th configuration from offset rank); with
    world * n == total the ranks cover the sweep exactly once."""
    tot = n * world
    return [((rank + world * j) * total) // tot for j in range(n)]


def cfg5_instances(idx, T: int = 288, K: int = 100):
    """Instances idx of the cfg5 sweep: cfg2's price chain (shared lambda, P), pbar/delta in [10.42, 99]
    (8 h down to 0.84 h at 5-min stages), eta_c = eta_d in [0.80, 0.99]; sbar/delta = 1000."""
    sweep = cfg5_sweep()
    base = cfg2(T=T, K=K)
    out = []
    for j in idx:
        c = sweep[j % len(sweep)]
        out.append(Instance(f"cfg5[{j}]", T, K, c["pbar"], 1000.0, 500.0, c["eta"], c["eta"], 1.0, base.lam, base.P,
                            base.pi, meta=dict(sweep_index=j)))
    return out


# ---------------------------------------------------------------------------------------------
# Random small instances for parity / pin tests
# ---------------------------------------------------------------------------------------------

def random_instance(seed: int, T: int | None = None, K: int | None = None, S_max: int = 12,
                    rank1: bool | None = None, payoff: int | None = None, lattice: bool = False,
                    neg_prices: bool = False) -> Instance:
    """A seeded random problem with small sizes.  lattice=True keeps every action on the state
    lattice (eta = 1, integral pbar/delta) so no interpolation occurs."""
    rng = np.random.Generator(np.random.PCG64(seed))
    T = T if T is not None else int(rng.integers(1, 6))
    K = K if K is not None else int(rng.integers(1, 4))
    delta = float(rng.choice([0.5, 1.0, 0.25]))
    ns = int(rng.integers(2, S_max))
    sbar = ns * delta
    if lattice:
        eta_c = eta_d = 1.0
        pbar = float(rng.integers(1, max(2, ns))) * delta
    else:
        eta_c = float(rng.uniform(0.7, 1.0)); eta_d = float(rng.uniform(0.7, 1.0))
        pbar = float(rng.uniform(0.6, max(0.7, 0.8 * ns))) * delta
    s0 = float(rng.integers(0, ns + 1)) * delta
    lam = rng.normal(30.0, 20.0, size=(T, K))
    if neg_prices:
        lam = lam - lam.max()
    if rank1 is None:
        rank1 = bool(rng.integers(0, 2))
    if rank1:
        P = None
        pi = rng.dirichlet(np.ones(K), size=T)
    else:
        P = rng.dirichlet(np.ones(K), size=(max(T - 1, 0), K)) if T > 1 else np.zeros((0, K, K))
        pi = rng.dirichlet(np.ones(K))
    payoff = payoff if payoff is not None else PAYOFF_LINEAR
    return Instance(f"rand{seed}", T, K, pbar, sbar, s0, eta_c, eta_d, delta, np.ascontiguousarray(lam),
                    None if P is None else np.ascontiguousarray(P), np.ascontiguousarray(pi),
                    None, payoff, None, dict(seed=seed))


def random_g(seed: int, A: int, scale: float = 5.0) -> np.ndarray:
    rng = np.random.Generator(np.random.PCG64(seed + 777))
    return rng.uniform(0.0, scale, size=A)


def random_table(seed: int, T: int, K: int, A: int) -> np.ndarray:
    rng = np.random.Generator(np.random.PCG64(seed + 999))
    return rng.normal(0.0, 10.0, size=(T, K, A))
