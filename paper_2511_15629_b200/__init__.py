"""Python binding of libesdp.so (include/esdp.h): argument marshalling only.

Every step of the method runs in the CUDA kernels behind the C ABI; this module converts numpy
arrays / torch tensors into the C structs and pointers and raises on a non-OK status.  There is
no fallback: if libesdp.so is missing or fails to load, importing this package raises.

The function names mirror the C ABI (esdp_create, esdp_backward, ...).  ``Solver`` is a small
owning wrapper around one context.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

__all__ = [
    "ESDP_OK", "ESDP_E_CONFIG", "ESDP_E_DATA", "ESDP_E_INTERNAL", "ESDP_E_STATE", "ESDP_E_CUDA",
    "ESDP_E_NCCL", "ESDP_E_NOMEM", "ESDP_PAYOFF_LINEAR", "ESDP_PAYOFF_LINEAR_MINUS_G",
    "ESDP_PAYOFF_TABLE", "ESDP_KEEP_VALUES", "EsdpError", "esdp_problem", "LIB_PATH", "lib",
    "esdp_create", "esdp_dims", "esdp_actions", "esdp_load", "esdp_load_async", "esdp_backward", "esdp_backward_async",
    "esdp_objective", "esdp_values", "esdp_policy", "esdp_bidcurves", "esdp_bidcurves_dev",
    "esdp_simulate", "esdp_simulate_dev", "esdp_launch_count", "esdp_kernel_times", "esdp_destroy",
    "esdp_last_error", "ESDP_PROFILE", "ESDP_FORCE_BRUTE", "esdp_stencil_kind", "Solver", "Batch", "EXPORTED_SYMBOLS",
]

ESDP_OK, ESDP_E_CONFIG, ESDP_E_DATA, ESDP_E_INTERNAL, ESDP_E_STATE, ESDP_E_CUDA, ESDP_E_NCCL, ESDP_E_NOMEM = range(8)
ESDP_PAYOFF_LINEAR, ESDP_PAYOFF_LINEAR_MINUS_G, ESDP_PAYOFF_TABLE = 0, 1, 2
ESDP_KEEP_VALUES = 1
ESDP_PROFILE = 2
ESDP_FORCE_BRUTE = 4
ESDP_NO_PDL = 8
ESDP_NO_DMMA = 16
ESDP_CONTRACT_OZAKI = 32
ESDP_FLAGS_ALL = 63
ESDP_SIM_LOTTERY, ESDP_SIM_PHYSICAL, ESDP_SIM_CLEAR_BIDS, ESDP_SIM_SELF, ESDP_SIM_FIXED = 0, 1, 2, 3, 4

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libesdp.so")

EXPORTED_SYMBOLS = [
    "esdp_create", "esdp_dims", "esdp_actions", "esdp_load", "esdp_load_async", "esdp_backward", "esdp_backward_async",
    "esdp_objective", "esdp_values", "esdp_policy", "esdp_bidcurves", "esdp_bidcurves_dev",
    "esdp_simulate", "esdp_simulate_dev", "esdp_launch_count", "esdp_kernel_times", "esdp_stencil_kind",
    "esdp_debug_time", "esdp_window_fallbacks", "esdp_window_level_tables", "esdp_destroy", "esdp_last_error",
    "esdp_create_dist", "esdp_nccl_unique_id", "esdp_partition", "esdp_dist_info", "esdp_set_bid_requests",
    "esdp_simulate_mode", "esdp_simulate_mode_dev", "esdp_simulate_strategy_dev", "esdp_price_paths_dev",
    "esdp_simulate_async", "esdp_objective_async",
    "esdp_create_batch", "esdp_batch_dims", "esdp_batch_backward", "esdp_batch_backward_async",
    "esdp_batch_objective", "esdp_batch_policy", "esdp_batch_value1", "esdp_batch_simulate_dev",
    "esdp_batch_launch_count", "esdp_batch_destroy", "esdp_batch_last_error", "esdp_batch_load_async",
    "esdp_batch_kernel_time", "esdp_batch_plan", "esdp_expectation_dev",
]

_dp = ctypes.POINTER(ctypes.c_double)
_i32p = ctypes.POINTER(ctypes.c_int32)
_i16p = ctypes.POINTER(ctypes.c_int16)
_vp = ctypes.c_void_p


class esdp_problem(ctypes.Structure):
    _fields_ = [
        ("T", ctypes.c_int32), ("K", ctypes.c_int32),
        ("pbar", ctypes.c_double), ("sbar", ctypes.c_double), ("s0", ctypes.c_double),
        ("eta_c", ctypes.c_double), ("eta_d", ctypes.c_double), ("delta", ctypes.c_double),
        ("A", ctypes.c_int32), ("actions", _dp),
        ("lambda_", _dp), ("P", _dp), ("pi", _dp),
        ("payoff_kind", ctypes.c_int32), ("g", _dp),
        ("flags", ctypes.c_uint32),
    ]


class EsdpError(RuntimeError):
    def __init__(self, status: int, what: str, msg: str):
        super().__init__(f"{what} failed with status {status}: {msg}")
        self.status = status


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libesdp.so not found at {LIB_PATH}; build it with `make` (or __graft_entry__.build())")
    L = ctypes.CDLL(LIB_PATH)
    ctx = _vp
    sig = {
        "esdp_create": ([ctypes.POINTER(esdp_problem), ctypes.POINTER(_vp)], ctypes.c_int),
        "esdp_dims": ([ctx, _i32p, _i32p, _i32p, _i32p], ctypes.c_int),
        "esdp_actions": ([ctx, _dp], ctypes.c_int),
        "esdp_load": ([ctx, _dp, _dp, _dp, _dp], ctypes.c_int),
        "esdp_load_async": ([ctx, _dp, _dp, _dp, _dp], ctypes.c_int),
        "esdp_backward": ([ctx, _vp, _dp], ctypes.c_int),
        "esdp_backward_async": ([ctx, _vp], ctypes.c_int),
        "esdp_objective": ([ctx, _dp], ctypes.c_int),
        "esdp_objective_async": ([ctx, _vp, _vp], ctypes.c_int),
        "esdp_simulate_async": ([ctx, ctypes.c_int64, ctypes.c_uint64, _vp, _vp], ctypes.c_int),
        "esdp_values": ([ctx, ctypes.c_int32, _dp, _dp], ctypes.c_int),
        "esdp_policy": ([ctx, ctypes.c_int32, _i16p], ctypes.c_int),
        "esdp_bidcurves": ([ctx, ctypes.c_int64, _i32p, ctypes.c_int32, _i32p, _i16p, _dp, _dp], ctypes.c_int),
        "esdp_bidcurves_dev": ([ctx, ctypes.c_int64, _vp, ctypes.c_int32, _vp, _vp, _vp, _vp, _vp], ctypes.c_int),
        "esdp_simulate": ([ctx, ctypes.c_int64, ctypes.c_uint64, _dp, _dp, _dp], ctypes.c_int),
        "esdp_simulate_dev": ([ctx, ctypes.c_int64, ctypes.c_uint64, _vp, _vp], ctypes.c_int),
        "esdp_simulate_mode": ([ctx, ctypes.c_int64, ctypes.c_uint64, ctypes.c_int32, _dp, _dp, _dp], ctypes.c_int),
        "esdp_simulate_mode_dev": ([ctx, ctypes.c_int64, ctypes.c_uint64, ctypes.c_int32, _vp, _vp], ctypes.c_int),
        "esdp_simulate_strategy_dev": ([ctx, ctypes.c_int64, ctypes.c_uint64, ctypes.c_int32, _vp, _vp, _vp, _vp],
                                       ctypes.c_int),
        "esdp_price_paths_dev": ([ctx, ctypes.c_int64, ctypes.c_uint64, _vp, _vp, _vp], ctypes.c_int),
        "esdp_launch_count": ([ctx, ctypes.POINTER(ctypes.c_int64)], ctypes.c_int),
        "esdp_kernel_times": ([ctx, _dp, _dp], ctypes.c_int),
        "esdp_stencil_kind": ([ctx, _i32p], ctypes.c_int),
        "esdp_debug_time": ([ctx, ctypes.c_int32, ctypes.c_int32, _dp], ctypes.c_int),
        "esdp_window_fallbacks": ([ctx, ctypes.POINTER(ctypes.c_int64)], ctypes.c_int),
        "esdp_window_level_tables": ([ctx, ctypes.POINTER(ctypes.c_int64)], ctypes.c_int),
        "esdp_create_dist": ([ctypes.POINTER(esdp_problem), ctypes.c_int32, ctypes.c_int32, ctypes.c_char_p,
                              ctypes.POINTER(_vp)], ctypes.c_int),
        "esdp_nccl_unique_id": ([ctypes.c_char_p], ctypes.c_int),
        "esdp_dist_info": ([ctx, _i32p, _i32p, _i32p], ctypes.c_int),
        "esdp_set_bid_requests": ([ctx, ctypes.c_int64, _i32p, ctypes.c_int32, _vp, _vp, _vp, _vp], ctypes.c_int),
        "esdp_partition": ([ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, _i32p, _i32p, _i32p], ctypes.c_int),
        "esdp_destroy": ([ctx], None),
        "esdp_last_error": ([ctx], ctypes.c_char_p),
        "esdp_create_batch": ([ctypes.POINTER(esdp_problem), ctypes.c_int32, ctypes.POINTER(_vp)], ctypes.c_int),
        "esdp_batch_dims": ([ctx, _i32p, _i32p, _i32p, _i32p, _i32p], ctypes.c_int),
        "esdp_batch_backward": ([ctx, _vp, _dp], ctypes.c_int),
        "esdp_batch_backward_async": ([ctx, _vp], ctypes.c_int),
        "esdp_batch_objective": ([ctx, _dp], ctypes.c_int),
        "esdp_batch_policy": ([ctx, ctypes.c_int32, ctypes.c_int32, _i16p], ctypes.c_int),
        "esdp_batch_value1": ([ctx, ctypes.c_int32, _dp], ctypes.c_int),
        "esdp_batch_simulate_dev": ([ctx, ctypes.c_int64, ctypes.c_uint64, _vp, _vp], ctypes.c_int),
        "esdp_batch_launch_count": ([ctx, ctypes.POINTER(ctypes.c_int64)], ctypes.c_int),
        "esdp_batch_load_async": ([ctx, _vp, _vp, _vp, _vp], ctypes.c_int),
        "esdp_batch_kernel_time": ([ctx, ctypes.c_int32, ctypes.c_int32, _dp], ctypes.c_int),
        "esdp_batch_plan": ([ctx, _i32p], ctypes.c_int),
        "esdp_expectation_dev": ([_vp, _vp, _vp, ctypes.c_int32, ctypes.c_int32, ctypes.c_int64, ctypes.c_int64,
                                  ctypes.c_int64, ctypes.c_int32, _vp], ctypes.c_int),
        "esdp_batch_destroy": ([ctx], None),
        "esdp_batch_last_error": ([ctx], ctypes.c_char_p),
    }
    for name, (args, res) in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = res
    return L


lib = _load()


def _p(a, t=_dp):
    return None if a is None else a.ctypes.data_as(t)


def _f64(a):
    return None if a is None else np.ascontiguousarray(a, dtype=np.float64)


def esdp_last_error(ctx=None) -> str:
    m = lib.esdp_last_error(ctx)
    return m.decode() if m else ""


def _check(st, what, ctx=None):
    if st != ESDP_OK:
        raise EsdpError(st, what, esdp_last_error(ctx))


def esdp_create(T, K, pbar, sbar, s0, eta_c, eta_d, delta, lam, P, pi, actions=None,
                payoff_kind=ESDP_PAYOFF_LINEAR, g=None, flags=0, dist=None):
    """esdp_create(&problem, &ctx) -> opaque context handle (int).
    dist = (world, rank, nccl_id_bytes) selects esdp_create_dist (multi-GPU, K-partitioned)."""
    keep = [_f64(x) for x in (actions, lam, P, pi, g)]
    act, lam_, P_, pi_, g_ = keep
    pr = esdp_problem(int(T), int(K), float(pbar), float(sbar), float(s0), float(eta_c), float(eta_d),
                      float(delta), 0 if act is None else int(act.shape[0]), _p(act), _p(lam_), _p(P_),
                      _p(pi_), int(payoff_kind), _p(g_), int(flags))
    out = _vp()
    if dist is None:
        st = lib.esdp_create(ctypes.byref(pr), ctypes.byref(out))
        _check(st, "esdp_create", None)
    else:
        world, rank, nid = dist
        st = lib.esdp_create_dist(ctypes.byref(pr), int(world), int(rank), bytes(nid), ctypes.byref(out))
        _check(st, "esdp_create_dist", None)
    return out.value


def esdp_create_dist(world, rank, nccl_id, *args, **kw):
    """Multi-GPU context: this rank owns the price-state rows esdp_partition(K, world, rank)."""
    return esdp_create(*args, dist=(world, rank, nccl_id), **kw)


def esdp_nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(lib.esdp_nccl_unique_id(buf), "esdp_nccl_unique_id", None)
    return buf.raw


def esdp_dist_info(ctx):
    """(world, rank, nccl_nranks) of a context; nccl_nranks is the communicator's ncclCommCount (0: none)."""
    w, r, n = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
    _check(lib.esdp_dist_info(ctx, ctypes.byref(w), ctypes.byref(r), ctypes.byref(n)), "esdp_dist_info", ctx)
    return w.value, r.value, n.value


def esdp_partition(K, world, rank):
    """(k_lo, k_cnt, kmax): the rows [k_lo, k_lo + k_cnt) owned by `rank` (host-only, no GPU)."""
    lo, cnt, m = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
    _check(lib.esdp_partition(int(K), int(world), int(rank), ctypes.byref(lo), ctypes.byref(cnt), ctypes.byref(m)),
           "esdp_partition", None)
    return lo.value, cnt.value, m.value


def esdp_dims(ctx):
    T, S, A, K = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
    _check(lib.esdp_dims(ctx, ctypes.byref(T), ctypes.byref(S), ctypes.byref(A), ctypes.byref(K)), "esdp_dims", ctx)
    return T.value, S.value, A.value, K.value


def esdp_actions(ctx):
    _, _, A, _ = esdp_dims(ctx)
    out = np.zeros(A)
    _check(lib.esdp_actions(ctx, _p(out)), "esdp_actions", ctx)
    return out


def esdp_load(ctx, lam=None, P=None, pi=None, g=None):
    keep = [_f64(x) for x in (lam, P, pi, g)]
    _check(lib.esdp_load(ctx, *[_p(x) for x in keep]), "esdp_load", ctx)


def esdp_load_async(ctx, lam=None, P=None, pi=None, g=None):
    """Validate and enqueue the upload; returns the host arrays, which the caller must keep alive (and
    unmodified) until the next backward pass has completed."""
    keep = [_f64(x) for x in (lam, P, pi, g)]
    _check(lib.esdp_load_async(ctx, *[_p(x) for x in keep]), "esdp_load_async", ctx)
    return keep


def _stream_ptr(stream):
    if stream is None:
        return None
    return getattr(stream, "cuda_stream", stream)


def esdp_backward(ctx, stream=None) -> float:
    J = ctypes.c_double()
    _check(lib.esdp_backward(ctx, _stream_ptr(stream), ctypes.byref(J)), "esdp_backward", ctx)
    return J.value


def esdp_backward_async(ctx, stream=None):
    _check(lib.esdp_backward_async(ctx, _stream_ptr(stream)), "esdp_backward_async", ctx)


def esdp_objective(ctx) -> float:
    J = ctypes.c_double()
    _check(lib.esdp_objective(ctx, ctypes.byref(J)), "esdp_objective", ctx)
    return J.value


def esdp_values(ctx, t, want_W=True):
    T, S, A, K = esdp_dims(ctx)
    V = np.zeros((K, S))
    W = np.zeros((K, S)) if want_W else None
    _check(lib.esdp_values(ctx, int(t), _p(V), _p(W)), "esdp_values", ctx)
    return (V, W) if want_W else V


def esdp_policy(ctx, t):
    T, S, A, K = esdp_dims(ctx)
    pol = np.zeros((K, S), np.int16)
    _check(lib.esdp_policy(ctx, int(t), _p(pol, _i16p)), "esdp_policy", ctx)
    return pol


def esdp_bidcurves(ctx, req, cap=None):
    """req: int array [n][3] of (t, i, k).  Returns dict(nvert, vert, q, price) (padded rows)."""
    T, S, A, K = esdp_dims(ctx)
    cap = A if cap is None else int(cap)
    req = np.ascontiguousarray(req, dtype=np.int32).reshape(-1, 3)
    n = req.shape[0]
    nv = np.zeros(n, np.int32)
    vert = np.zeros((n, cap), np.int16)
    q = np.zeros((n, cap))
    price = np.zeros((n, cap))
    _check(lib.esdp_bidcurves(ctx, n, _p(req, _i32p), cap, _p(nv, _i32p), _p(vert, _i16p), _p(q), _p(price)),
           "esdp_bidcurves", ctx)
    return dict(nvert=nv, vert=vert, q=q, price=price)


def esdp_bidcurves_dev(ctx, n, req_ptr, cap, nvert_ptr, vert_ptr, q_ptr, price_ptr, stream=None):
    _check(lib.esdp_bidcurves_dev(ctx, int(n), req_ptr, int(cap), nvert_ptr, vert_ptr, q_ptr, price_ptr,
                                  _stream_ptr(stream)), "esdp_bidcurves_dev", ctx)


def esdp_set_bid_requests(ctx, req, cap, nvert_ptr, vert_ptr, q_ptr, price_ptr):
    """Bid curves extracted inside every following backward pass (device outputs, vertex-major)."""
    req = np.ascontiguousarray(req, dtype=np.int32).reshape(-1, 3)
    _check(lib.esdp_set_bid_requests(ctx, req.shape[0], _p(req, _i32p), int(cap), nvert_ptr, vert_ptr, q_ptr, price_ptr),
           "esdp_set_bid_requests", ctx)


def esdp_simulate(ctx, n_paths, seed, per_path=True):
    m, v = ctypes.c_double(), ctypes.c_double()
    out = np.zeros(int(n_paths)) if per_path else None
    _check(lib.esdp_simulate(ctx, int(n_paths), ctypes.c_uint64(int(seed)), ctypes.byref(m), ctypes.byref(v),
                             _p(out)), "esdp_simulate", ctx)
    return out, m.value, v.value


def esdp_simulate_mode(ctx, n_paths, seed, mode, per_path=True):
    m, v = ctypes.c_double(), ctypes.c_double()
    out = np.zeros(int(n_paths)) if per_path else None
    _check(lib.esdp_simulate_mode(ctx, int(n_paths), ctypes.c_uint64(int(seed)), int(mode), ctypes.byref(m),
                                  ctypes.byref(v), _p(out)), "esdp_simulate_mode", ctx)
    return out, m.value, v.value


def esdp_simulate_strategy_dev(ctx, n_paths, seed, mode, per_path_ptr, schedule_ptr=None, actions_ptr=None,
                               stream=None):
    _check(lib.esdp_simulate_strategy_dev(ctx, int(n_paths), ctypes.c_uint64(int(seed)), int(mode), schedule_ptr,
                                          actions_ptr, per_path_ptr, _stream_ptr(stream)),
           "esdp_simulate_strategy_dev", ctx)


def esdp_price_paths_dev(ctx, n_paths, seed, kpath_ptr=None, lambda_ptr=None, stream=None):
    _check(lib.esdp_price_paths_dev(ctx, int(n_paths), ctypes.c_uint64(int(seed)), kpath_ptr, lambda_ptr,
                                    _stream_ptr(stream)), "esdp_price_paths_dev", ctx)


def esdp_simulate_dev(ctx, n_paths, seed, per_path_ptr, stream=None):
    _check(lib.esdp_simulate_dev(ctx, int(n_paths), ctypes.c_uint64(int(seed)), per_path_ptr, _stream_ptr(stream)),
           "esdp_simulate_dev", ctx)


def esdp_launch_count(ctx) -> int:
    n = ctypes.c_int64()
    _check(lib.esdp_launch_count(ctx, ctypes.byref(n)), "esdp_launch_count", ctx)
    return n.value


def esdp_kernel_times(ctx):
    """(ms per contraction launch, ms per stencil launch) averaged over the sampled stages of the last
    backward pass (needs ESDP_PROFILE)."""
    a, b = ctypes.c_double(), ctypes.c_double()
    _check(lib.esdp_kernel_times(ctx, ctypes.byref(a), ctypes.byref(b)), "esdp_kernel_times", ctx)
    return a.value, b.value


def esdp_stencil_kind(ctx) -> int:
    """bit 0: 1 = exact sliding-window stencil, 0 = brute force."""
    k = ctypes.c_int32()
    _check(lib.esdp_stencil_kind(ctx, ctypes.byref(k)), "esdp_stencil_kind", ctx)
    return k.value


def esdp_debug_time(ctx, what, reps=200) -> float:
    """Warm per-launch device time (us) of one kernel kind (0 contraction, 1 stencil, 2 brute stencil, 3 objective)."""
    us = ctypes.c_double()
    _check(lib.esdp_debug_time(ctx, int(what), int(reps), ctypes.byref(us)), "esdp_debug_time", ctx)
    return us.value


def esdp_window_level_tables(ctx) -> int:
    """Window-stencil run tables that were not unimodal (sparse-table levels built) since the last call."""
    n = ctypes.c_int64()
    _check(lib.esdp_window_level_tables(ctx, ctypes.byref(n)), "esdp_window_level_tables", ctx)
    return n.value


def esdp_window_fallbacks(ctx) -> int:
    """Rows re-scanned canonically by the window stencil since the last call (resets the counter)."""
    n = ctypes.c_int64()
    _check(lib.esdp_window_fallbacks(ctx, ctypes.byref(n)), "esdp_window_fallbacks", ctx)
    return n.value


def esdp_destroy(ctx):
    lib.esdp_destroy(ctx)


class Solver:
    """Owning wrapper of one esdp context.  `inst` is any object with the esdp_problem fields
    (T, K, pbar, sbar, s0, eta_c, eta_d, delta, lam, P, pi, actions, payoff_kind, g)."""

    def __init__(self, inst, keep_values=True, profile=False, force_brute=False, pdl=True, dmma=True,
                 dist=None):
        self.ctx = esdp_create(inst.T, inst.K, inst.pbar, inst.sbar, inst.s0, inst.eta_c, inst.eta_d, inst.delta,
                               inst.lam, inst.P, inst.pi, getattr(inst, "actions", None),
                               getattr(inst, "payoff_kind", ESDP_PAYOFF_LINEAR), getattr(inst, "g", None),
                               (ESDP_KEEP_VALUES if keep_values else 0) | (ESDP_PROFILE if profile else 0)
                               | (ESDP_FORCE_BRUTE if force_brute else 0) | (0 if pdl else ESDP_NO_PDL)
                               | (0 if dmma else ESDP_NO_DMMA), dist=dist)
        self.T, self.S, self.A, self.K = esdp_dims(self.ctx)
        self.stencil_kind = esdp_stencil_kind(self.ctx)

    def backward(self, stream=None):
        return esdp_backward(self.ctx, stream)

    def values(self, t, want_W=True):
        return esdp_values(self.ctx, t, want_W)

    def policy(self, t):
        return esdp_policy(self.ctx, t)

    def actions(self):
        return esdp_actions(self.ctx)

    def bidcurves(self, req, cap=None):
        return esdp_bidcurves(self.ctx, req, cap)

    def simulate(self, n_paths, seed, per_path=True, mode=ESDP_SIM_LOTTERY):
        if mode == ESDP_SIM_LOTTERY:
            return esdp_simulate(self.ctx, n_paths, seed, per_path)
        return esdp_simulate_mode(self.ctx, n_paths, seed, mode, per_path)

    def close(self):
        if self.ctx:
            esdp_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


class Batch:
    """A batch of instances sharing one price model (esdp_create_batch, cfg5): one graph for all."""

    def __init__(self, insts, force_brute=False, ozaki=False):
        keep = []
        probs = (esdp_problem * len(insts))()
        for j, inst in enumerate(insts):   # every instance's own arrays: the library checks they match
            act = _f64(getattr(inst, "actions", None))
            g = _f64(getattr(inst, "g", None))
            lam, P, pi = _f64(inst.lam), _f64(inst.P), _f64(inst.pi)
            keep += [act, g, lam, P, pi]
            probs[j] = esdp_problem(int(inst.T), int(inst.K), float(inst.pbar), float(inst.sbar), float(inst.s0),
                                    float(inst.eta_c), float(inst.eta_d), float(inst.delta),
                                    0 if act is None else int(act.shape[0]), _p(act), _p(lam), _p(P), _p(pi),
                                    int(getattr(inst, "payoff_kind", ESDP_PAYOFF_LINEAR)), _p(g),
                                    (ESDP_FORCE_BRUTE if (force_brute[j] if isinstance(force_brute, (list, tuple))
                                                          else force_brute) else 0) |
                                    (ESDP_CONTRACT_OZAKI if ozaki else 0))
        out = _vp()
        st = lib.esdp_create_batch(probs, len(insts), ctypes.byref(out))
        if st != ESDP_OK:
            m = lib.esdp_batch_last_error(None)
            raise EsdpError(st, "esdp_create_batch", m.decode() if m else "")
        self.b = out.value
        n, T, S, K = (ctypes.c_int32() for _ in range(4))
        A = (ctypes.c_int32 * len(insts))()
        lib.esdp_batch_dims(self.b, ctypes.byref(n), ctypes.byref(T), ctypes.byref(S), ctypes.byref(K), A)
        self.n, self.T, self.S, self.K = n.value, T.value, S.value, K.value
        self.A = list(A)

    def _check(self, st, what):
        if st != ESDP_OK:
            m = lib.esdp_batch_last_error(self.b)
            raise EsdpError(st, what, m.decode() if m else "")

    def backward(self, stream=None):
        J = np.zeros(self.n)
        self._check(lib.esdp_batch_backward(self.b, _stream_ptr(stream), _p(J)), "esdp_batch_backward")
        return J

    def backward_async(self, stream=None):
        self._check(lib.esdp_batch_backward_async(self.b, _stream_ptr(stream)), "esdp_batch_backward_async")

    def objective(self):
        J = np.zeros(self.n)
        self._check(lib.esdp_batch_objective(self.b, _p(J)), "esdp_batch_objective")
        return J

    def policy(self, m, t):
        out = np.zeros((self.K, self.S), np.int16)
        self._check(lib.esdp_batch_policy(self.b, int(m), int(t), _p(out, _i16p)), "esdp_batch_policy")
        return out

    def value1(self, m):
        out = np.zeros((self.K, self.S))
        self._check(lib.esdp_batch_value1(self.b, int(m), _p(out)), "esdp_batch_value1")
        return out

    def simulate_dev(self, n_paths, seed, out_ptr, stream=None):
        self._check(lib.esdp_batch_simulate_dev(self.b, int(n_paths), ctypes.c_uint64(int(seed)), out_ptr,
                                                _stream_ptr(stream)), "esdp_batch_simulate_dev")

    def launch_count(self):
        n = ctypes.c_int64()
        self._check(lib.esdp_batch_launch_count(self.b, ctypes.byref(n)), "esdp_batch_launch_count")
        return n.value

    def load_async(self, lam_ptr, P_ptr, pi_ptr, stream=None):
        """esdp_batch_load_async from host addresses (pinned buffers: keep them alive until the stream passes)."""
        self._check(lib.esdp_batch_load_async(self.b, lam_ptr, P_ptr, pi_ptr, _stream_ptr(stream)), "esdp_batch_load_async")

    def kernel_time(self, what, reps=100):
        us = ctypes.c_double()
        self._check(lib.esdp_batch_kernel_time(self.b, int(what), int(reps), ctypes.byref(us)), "esdp_batch_kernel_time")
        return us.value

    @property
    def plan(self):
        """Expectation plan (esdp_batch_plan): 0 FP64 DMMA, 1 DFMA, 2 Ozaki u8 tcgen05."""
        v = ctypes.c_int32()
        self._check(lib.esdp_batch_plan(self.b, ctypes.byref(v)), "esdp_batch_plan")
        return v.value

    def close(self):
        if self.b:
            lib.esdp_batch_destroy(self.b)
            self.b = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def expectation_dev(P_ptr, V_ptr, W_ptr, rows, K, ncols, ldv, ldw, method, stream=None):
    """esdp_expectation_dev: W = P V on device buffers (method 0 canonical DMMA chain, 1 Ozaki u8 tcgen05)."""
    st = lib.esdp_expectation_dev(P_ptr, V_ptr, W_ptr, int(rows), int(K), int(ncols), int(ldv), int(ldw), int(method),
                                  stream)
    if st != ESDP_OK:
        m = lib.esdp_batch_last_error(None)
        raise EsdpError(st, "esdp_expectation_dev", m.decode() if m else "")
