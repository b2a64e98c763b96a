"""Small test helpers: convert workloads.Instance into the oracle's Problem / the product's problem."""
from __future__ import annotations

import numpy as np

import oracle


def to_oracle(inst) -> oracle.Problem:
    return oracle.Problem(T=inst.T, K=inst.K, pbar=inst.pbar, sbar=inst.sbar, s0=inst.s0,
                          eta_c=inst.eta_c, eta_d=inst.eta_d, delta=inst.delta, lam=inst.lam,
                          P=inst.P, pi=inst.pi, actions=inst.actions, payoff_kind=inst.payoff_kind,
                          g=inst.g)


def simple_problem(pbar, sbar, delta, eta, eta_d=None, T=1, K=1, lam=None, s0=0.0) -> oracle.Problem:
    """Deterministic (K = 1 unless asked) problem with given prices."""
    eta_d = eta if eta_d is None else eta_d
    if lam is None:
        lam = np.zeros((T, K))
    lam = np.asarray(lam, dtype=np.float64).reshape(T, K)
    P = np.full((max(T - 1, 0), K, K), 1.0 / K)
    pi = np.full(K, 1.0 / K)
    return oracle.Problem(T=T, K=K, pbar=pbar, sbar=sbar, s0=s0, eta_c=eta, eta_d=eta_d, delta=delta,
                          lam=lam, P=P, pi=pi)


def rel_err(a, b):
    a = np.asarray(a, dtype=np.float64); b = np.asarray(b, dtype=np.float64)
    den = np.maximum(np.maximum(np.abs(a), np.abs(b)), 1e-300)
    d = np.abs(a - b)
    d = np.where(a == b, 0.0, d)
    return float(np.max(d / np.maximum(den, 1.0))) if d.size else 0.0
