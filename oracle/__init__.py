"""ctypes front end of the FP64 CPU oracle (oracle/esdp_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs.  The product (CUDA) package never
imports this module, and nothing here imports the product.

Arrays are numpy float64 / int16, C-contiguous; shapes follow esdp_oracle.h.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")

REF_OK, REF_E_CONFIG, REF_E_DATA, REF_E_INTERNAL, REF_E_STATE = 0, 1, 2, 3, 4
PAYOFF_LINEAR, PAYOFF_LINEAR_MINUS_G, PAYOFF_TABLE = 0, 1, 2

_dp = ctypes.POINTER(ctypes.c_double)
_ip = ctypes.POINTER(ctypes.c_int32)
_sp = ctypes.POINTER(ctypes.c_int16)


class _Problem(ctypes.Structure):
    _fields_ = [
        ("T", ctypes.c_int32), ("K", ctypes.c_int32),
        ("pbar", ctypes.c_double), ("sbar", ctypes.c_double), ("s0", ctypes.c_double),
        ("eta_c", ctypes.c_double), ("eta_d", ctypes.c_double), ("delta", ctypes.c_double),
        ("A", ctypes.c_int32), ("actions", _dp),
        ("lam", _dp), ("P", _dp), ("pi", _dp),
        ("payoff_kind", ctypes.c_int32), ("g", _dp),
    ]


def build(force: bool = False) -> str:
    """Compile liboracle.so with plain gcc (no -ffast-math, no FMA contraction)."""
    src = os.path.join(_HERE, "esdp_oracle.c")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        cmd = (f"gcc -O2 -std=c11 -ffp-contract=off -fno-fast-math -fopenmp -fPIC -shared "
               f"-o {_LIB_PATH} {src} -lm")
        rc = os.system(cmd)
        if rc != 0:
            raise RuntimeError(f"oracle build failed: {cmd}")
    return _LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB_PATH)
        P = ctypes.POINTER(_Problem)
        L.ref_dims.argtypes = [P, _ip, _ip]
        L.ref_actions.argtypes = [P, _dp]
        L.ref_tables.argtypes = [P, _ip, _dp, _dp, _ip, _ip]
        L.ref_backward.argtypes = [P, ctypes.c_int32, ctypes.c_int32, _dp, _dp, _sp, _dp]
        L.ref_bidcurve.argtypes = [P, _dp, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                   ctypes.c_int32, _ip, _sp, _dp, _dp, _ip]
        L.ref_clear.argtypes = [ctypes.c_int32, _dp, ctypes.c_double]
        L.ref_clear.restype = ctypes.c_int32
        L.ref_philox4x32_10.argtypes = [ctypes.POINTER(ctypes.c_uint32), ctypes.POINTER(ctypes.c_uint32),
                                        ctypes.POINTER(ctypes.c_uint32)]
        L.ref_simulate.argtypes = [P, _sp, ctypes.c_int64, ctypes.c_uint64, _dp, _dp, _dp]
        L.ref_simulate_mode.argtypes = [P, _sp, _dp, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, _dp, _dp, _dp]
        L.ref_simulate_strategy.argtypes = [P, _dp, ctypes.c_int32, _sp, ctypes.c_int64, ctypes.c_uint64, _dp, _sp]
        L.ref_stage.argtypes = [P, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, _dp, _dp, _dp, _sp]
        L.ref_objective.argtypes = [P, _dp, _dp]
        _lib = L
    return _lib


def _ptr(a, t=_dp):
    return None if a is None else a.ctypes.data_as(t)


class OracleError(RuntimeError):
    def __init__(self, code, what):
        super().__init__(f"{what}: oracle status {code}")
        self.code = code


@dataclass
class Problem:
    """Problem statement in the oracle's terms."""
    T: int
    K: int
    pbar: float
    sbar: float
    s0: float
    eta_c: float
    eta_d: float
    delta: float
    lam: np.ndarray                 # [T][K]
    P: np.ndarray | None            # [T-1][K][K] or None (rank-1)
    pi: np.ndarray                  # [K] or [T][K]
    actions: np.ndarray | None = None
    payoff_kind: int = PAYOFF_LINEAR
    g: np.ndarray | None = None

    def _c(self):
        self._keep = [np.ascontiguousarray(x, dtype=np.float64) if x is not None else None
                      for x in (self.actions, self.lam, self.P, self.pi, self.g)]
        act, lam, P, pi, g = self._keep
        return _Problem(int(self.T), int(self.K), float(self.pbar), float(self.sbar), float(self.s0),
                        float(self.eta_c), float(self.eta_d), float(self.delta),
                        0 if act is None else int(act.shape[0]), _ptr(act),
                        _ptr(lam), _ptr(P), _ptr(pi), int(self.payoff_kind), _ptr(g))


def dims(pr: Problem):
    c = pr._c()
    S, A = ctypes.c_int32(), ctypes.c_int32()
    rc = lib().ref_dims(ctypes.byref(c), ctypes.byref(S), ctypes.byref(A))
    if rc:
        raise OracleError(rc, "ref_dims")
    return S.value, A.value


def status_of(pr: Problem) -> int:
    c = pr._c()
    S, A = ctypes.c_int32(), ctypes.c_int32()
    return lib().ref_dims(ctypes.byref(c), ctypes.byref(S), ctypes.byref(A))


def actions(pr: Problem) -> np.ndarray:
    S, A = dims(pr)
    out = np.zeros(A)
    c = pr._c()
    rc = lib().ref_actions(ctypes.byref(c), _ptr(out))
    if rc:
        raise OracleError(rc, "ref_actions")
    return out


def tables(pr: Problem):
    S, A = dims(pr)
    off = np.zeros(A, np.int32); w = np.zeros(A); omw = np.zeros(A)
    ilo = np.zeros(A, np.int32); ihi = np.zeros(A, np.int32)
    c = pr._c()
    rc = lib().ref_tables(ctypes.byref(c), _ptr(off, _ip), _ptr(w), _ptr(omw), _ptr(ilo, _ip), _ptr(ihi, _ip))
    if rc:
        raise OracleError(rc, "ref_tables")
    return dict(off=off, w=w, omw=omw, ilo=ilo, ihi=ihi)


@dataclass
class Solution:
    V: np.ndarray     # [T][K][S]
    W: np.ndarray     # [T][K][S]
    pol: np.ndarray   # [T][K][S] int16
    J: float | None


def backward(pr: Problem, t_stop: int = 1, nthreads: int = 1) -> Solution:
    S, A = dims(pr)
    V = np.zeros((pr.T, pr.K, S)); W = np.zeros((pr.T, pr.K, S))
    pol = np.full((pr.T, pr.K, S), -1, np.int16)
    J = ctypes.c_double(np.nan)
    c = pr._c()
    rc = lib().ref_backward(ctypes.byref(c), int(t_stop), int(nthreads), _ptr(V), _ptr(W),
                            _ptr(pol, _sp), ctypes.byref(J))
    if rc:
        raise OracleError(rc, "ref_backward")
    return Solution(V, W, pol, J.value if t_stop == 1 else None)


def stage(pr: Problem, t: int, k_lo: int, k_hi: int, Vnext, nthreads: int = 1):
    """Stage t for rows [k_lo, k_hi): returns (W rows, V rows, pol rows), each [k_hi-k_lo][S]."""
    S, A = dims(pr)
    n = k_hi - k_lo
    W = np.zeros((n, S)); V = np.zeros((n, S)); pol = np.full((n, S), -1, np.int16)
    Vn = None if Vnext is None else np.ascontiguousarray(Vnext, dtype=np.float64)
    c = pr._c()
    rc = lib().ref_stage(ctypes.byref(c), int(t), int(k_lo), int(k_hi), int(nthreads), _ptr(Vn), _ptr(W), _ptr(V),
                         _ptr(pol, _sp))
    if rc:
        raise OracleError(rc, "ref_stage")
    return W, V, pol


def objective(pr: Problem, V1) -> float:
    J = ctypes.c_double()
    V1 = np.ascontiguousarray(V1, dtype=np.float64)
    c = pr._c()
    rc = lib().ref_objective(ctypes.byref(c), _ptr(V1), ctypes.byref(J))
    if rc:
        raise OracleError(rc, "ref_objective")
    return J.value


def bidcurve(pr: Problem, W: np.ndarray, t: int, i: int, k: int):
    S, A = dims(pr)
    nv = ctypes.c_int32(); reps = ctypes.c_int32()
    vert = np.zeros(A, np.int16); q = np.zeros(A); price = np.zeros(max(A - 1, 1))
    c = pr._c()
    Wc = np.ascontiguousarray(W, dtype=np.float64)
    rc = lib().ref_bidcurve(ctypes.byref(c), _ptr(Wc), int(t), int(i), int(k), A, ctypes.byref(nv),
                            _ptr(vert, _sp), _ptr(q), _ptr(price), ctypes.byref(reps))
    if rc:
        raise OracleError(rc, "ref_bidcurve")
    n = nv.value
    return dict(nvert=n, vert=vert[:n].copy(), q=q[:n].copy(), price=price[:max(n - 1, 0)].copy(),
                repairs=reps.value)


def clear(curve, lam: float) -> int:
    pr = np.ascontiguousarray(curve["price"], dtype=np.float64)
    if pr.size == 0:
        pr = np.zeros(1)
    return lib().ref_clear(int(curve["nvert"]), _ptr(pr), float(lam))


def philox(ctr, key):
    c = (ctypes.c_uint32 * 4)(*ctr); k = (ctypes.c_uint32 * 2)(*key); o = (ctypes.c_uint32 * 4)()
    lib().ref_philox4x32_10(c, k, o)
    return [o[j] for j in range(4)]


def simulate(pr: Problem, pol: np.ndarray, n_paths: int, seed: int):
    per = np.zeros(n_paths)
    m = ctypes.c_double(); v = ctypes.c_double()
    c = pr._c()
    polc = np.ascontiguousarray(pol, dtype=np.int16)
    rc = lib().ref_simulate(ctypes.byref(c), _ptr(polc, _sp), int(n_paths), ctypes.c_uint64(seed),
                            _ptr(per), ctypes.byref(m), ctypes.byref(v))
    if rc:
        raise OracleError(rc, "ref_simulate")
    return per, m.value, v.value


SIM_LOTTERY, SIM_PHYSICAL, SIM_CLEAR_BIDS, SIM_SELF, SIM_FIXED = 0, 1, 2, 3, 4


def simulate_mode(pr: Problem, pol: np.ndarray, W: np.ndarray, mode: int, n_paths: int, seed: int):
    """ref_simulate_mode: lottery (pol), physical re-optimisation or bid clearing (W of every stage)."""
    per = np.zeros(n_paths)
    m = ctypes.c_double(); v = ctypes.c_double()
    c = pr._c()
    polc = np.ascontiguousarray(pol, dtype=np.int16)
    Wc = np.ascontiguousarray(W, dtype=np.float64)
    rc = lib().ref_simulate_mode(ctypes.byref(c), _ptr(polc, _sp), _ptr(Wc), int(mode), int(n_paths),
                                 ctypes.c_uint64(seed), _ptr(per), ctypes.byref(m), ctypes.byref(v))
    if rc:
        raise OracleError(rc, "ref_simulate_mode")
    return per, m.value, v.value


def simulate_strategy(pr: Problem, W, mode: int, n_paths: int, seed: int, schedule=None, want_actions=False):
    """ref_simulate_strategy: physical / self-scheduled / fixed-schedule dispatch; returns (profits,
    actions [T][n] or None)."""
    per = np.zeros(n_paths)
    c = pr._c()
    Wc = None if W is None else np.ascontiguousarray(W, dtype=np.float64)
    sch = None if schedule is None else np.ascontiguousarray(schedule, dtype=np.int16)
    act = np.zeros((pr.T, n_paths), np.int16) if want_actions else None
    rc = lib().ref_simulate_strategy(ctypes.byref(c), None if Wc is None else _ptr(Wc), int(mode),
                                     None if sch is None else _ptr(sch, _sp), int(n_paths), ctypes.c_uint64(seed),
                                     _ptr(per), None if act is None else _ptr(act, _sp))
    if rc:
        raise OracleError(rc, "ref_simulate_strategy")
    return per, act
