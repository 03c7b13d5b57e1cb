"""ctypes bindings for the oracle restatement (oracle/build/liboracle.so).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs -- never by the product
package.  Errors are raised as OracleError(code, message) with the codes of
toepfit_oracle.h (1 usage, 2 data, 3 numerical).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "build", "liboracle.so")

USAGE, DATA, NUMERICAL = 1, 2, 3


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


_lib = None

_f64p = C.POINTER(C.c_double)
_i64p = C.POINTER(C.c_int64)
_i32p = C.POINTER(C.c_int)


class LsarDiag(C.Structure):
    _fields_ = [
        ("fixed_idx", _i64p), ("fixed_w", _f64p),
        ("idx_out", _i64p), ("w_out", _f64p), ("rnorm2_out", _f64p), ("ssum_out", _f64p),
        ("scores_out", _f64p), ("resid_out", _f64p), ("scores_all", _f64p), ("method_out", _i32p),
    ]


class RhCfg(C.Structure):
    _fields_ = [("base_threshold", C.c_int64), ("sample_count", C.c_int64),
                ("gaussian_rows", C.c_int64), ("seed", C.c_uint64)]


class RhDiag(C.Structure):
    _fields_ = [
        ("fixed_idx", _i64p), ("fixed_w", _f64p),
        ("scores_out", _f64p), ("depth_out", _i32p), ("level_sizes", _i64p),
        ("level_idx", _i64p), ("level_idx_cap", C.c_int64),
        ("up_idx", _i64p), ("up_w", _f64p), ("idx_out", _i64p), ("w_out", _f64p),
        ("approx_out", _f64p), ("approx_rows", _i64p),
    ]


def build() -> None:
    subprocess.check_call(["make", "-s", "-C", HERE])


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = C.CDLL(LIB_PATH)
        L.orc_last_error.restype = C.c_char_p
        L.orc_mix.restype = C.c_uint64
        L.orc_mix.argtypes = [C.c_uint64]
        L.orc_derive_seed.restype = C.c_uint64
        L.orc_derive_seed.argtypes = [C.c_uint64, C.c_uint64]
        L.orc_default_base_threshold.restype = C.c_int64
        L.orc_default_base_threshold.argtypes = [C.c_int64, C.c_int64]
        L.orc_default_gaussian_rows.restype = C.c_int64
        L.orc_default_gaussian_rows.argtypes = [C.c_int64]
        L.orc_rh_time_upfront.restype = C.c_double
        L.orc_rh_time_upfront.argtypes = [_f64p, C.c_int64, C.c_int, C.c_int64, C.c_uint64]
        L.orc_lsar_time_one_lag.restype = C.c_double
        L.orc_lsar_time_one_lag.argtypes = [_f64p, C.c_int64, C.c_int, C.c_int64, C.c_int, C.c_uint64]
        L.orc_select_order.argtypes = [_f64p, C.c_int, C.c_double]
        _lib = L
    return _lib


def _p(a, t=_f64p):
    return a.ctypes.data_as(t) if a is not None else None


def _check(st: int) -> None:
    if st != 0:
        raise OracleError(st, lib().orc_last_error().decode())


def f64(x) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(x, dtype=np.float64))


def i64(x) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(x, dtype=np.int64))


def set_threads(n: int) -> None:
    lib().orc_set_threads(C.c_int(int(n)))


def max_threads() -> int:
    return int(lib().orc_max_threads())


# ---------------------------------------------------------------- RNG
def derive_seed(seed: int, tag: int) -> int:
    return int(lib().orc_derive_seed(C.c_uint64(seed), C.c_uint64(tag)))


class Rng:
    """rng.hpp:14-78 through the oracle."""

    def __init__(self, seed: int):
        self._s = (C.c_uint64 * 3)()
        self._st = C.create_string_buffer(24)
        lib().orc_rng_init(self._st, C.c_uint64(seed))
        lib().orc_rng_next.restype = C.c_uint64
        lib().orc_rng_uniform01.restype = C.c_double
        lib().orc_rng_normal.restype = C.c_double
        lib().orc_rng_below.restype = C.c_uint64
        lib().orc_rng_below.argtypes = [C.c_void_p, C.c_uint64]

    def __call__(self) -> int:
        return int(lib().orc_rng_next(self._st))

    def uniform01(self) -> float:
        return float(lib().orc_rng_uniform01(self._st))

    def normal(self) -> float:
        return float(lib().orc_rng_normal(self._st))

    def below(self, bound: int) -> int:
        return int(lib().orc_rng_below(self._st, bound))


# ---------------------------------------------------------------- primitives
def residuals(y, n_used: int, p: int, phi) -> np.ndarray:
    y = f64(y); phi = f64(phi)
    r = np.empty(n_used - p)
    _check(lib().orc_residuals(_p(y), C.c_int64(n_used), C.c_int(p), _p(phi), _p(r)))
    return r


def init_leverage_p1(window) -> np.ndarray:
    w = f64(window); out = np.empty_like(w)
    _check(lib().orc_init_leverage_p1(_p(w), C.c_int64(w.size), _p(out)))
    return out


def leverage_update(scores, r) -> np.ndarray:
    s = f64(scores); r = f64(r)
    if s.size != r.size:
        raise OracleError(USAGE, "score/residual length mismatch")
    out = np.empty_like(s)
    _check(lib().orc_leverage_update(_p(s), _p(r), C.c_int64(s.size), _p(out)))
    return out


def leverage_to_distribution(scores) -> np.ndarray:
    s = f64(scores); out = np.empty_like(s)
    _check(lib().orc_leverage_to_distribution(_p(s), C.c_int64(s.size), _p(out)))
    return out


def sample_rows(pi, c: int, seed: int):
    pi = f64(pi)
    idx = np.empty(max(c, 1), np.int64); w = np.empty(max(c, 1))
    _check(lib().orc_sample_rows(_p(pi), C.c_int64(pi.size), C.c_int64(c), C.c_uint64(seed),
                                 _p(idx, _i64p), _p(w)))
    return idx[:c], w[:c]


def apply_sample(y, n_used: int, p: int, idx, weights, width: int | None = None):
    y = f64(y); idx = i64(idx); weights = f64(weights)
    width = p if width is None else width
    c = idx.size
    a = np.empty((width, c)); b = np.empty(c)
    _check(lib().orc_apply_sample(_p(y), C.c_int64(n_used), C.c_int(p), _p(idx, _i64p),
                                  _p(weights), C.c_int64(c), C.c_int(width), _p(a), _p(b)))
    return a.T.copy(), b  # (c, width) row-major copy of the col-major matrix


def solve_exact(a, b):
    """Returns (x, method, rank); method 0 = CPQR, 1 = min-norm SVD."""
    a = np.asarray(a, dtype=np.float64)
    rows, cols = a.shape
    acm = np.asfortranarray(a)
    b = f64(b)
    x = np.empty(cols)
    method = C.c_int(0); rank = C.c_int64(0)
    _check(lib().orc_solve_exact(acm.ctypes.data_as(_f64p), C.c_int64(rows), C.c_int64(cols),
                                 _p(b), _p(x), C.byref(method), C.byref(rank)))
    return x, method.value, rank.value


def residual_norm_dd(a, b, x) -> float:
    """||a x - b|| in double-double (exact products, compensated sums)."""
    a = np.asfortranarray(np.asarray(a, dtype=np.float64))
    b = f64(b); x = f64(x)
    lib().orc_residual_norm_dd.restype = C.c_double
    return float(lib().orc_residual_norm_dd(a.ctypes.data_as(_f64p), C.c_int64(a.shape[0]), C.c_int64(a.shape[1]),
                                            _p(b), _p(x)))


def exact_leverage(a) -> np.ndarray:
    a = np.asarray(a, dtype=np.float64)
    rows, cols = a.shape
    acm = np.asfortranarray(a)
    out = np.empty(rows)
    _check(lib().orc_exact_leverage(acm.ctypes.data_as(_f64p), C.c_int64(rows), C.c_int64(cols),
                                    _p(out)))
    return out


def gaussian_apply(g: int, seed: int, m) -> np.ndarray:
    m = np.asfortranarray(np.asarray(m, dtype=np.float64))
    rows, cols = m.shape
    out = np.empty((cols, g))
    _check(lib().orc_gaussian_apply(C.c_int64(g), C.c_uint64(seed), m.ctypes.data_as(_f64p),
                                    C.c_int64(rows), C.c_int64(cols), _p(out)))
    return out.T.copy()


def generalized_leverage(cm, b, sketch_rows: int = 0, sketch_seed: int = 0) -> np.ndarray:
    cm = np.asfortranarray(np.asarray(cm, dtype=np.float64))
    b = np.asfortranarray(np.asarray(b, dtype=np.float64))
    if cm.shape[1] != b.shape[1]:
        raise OracleError(USAGE, "column count mismatch")
    out = np.empty(cm.shape[0])
    _check(lib().orc_generalized_leverage(cm.ctypes.data_as(_f64p), C.c_int64(cm.shape[0]),
                                          b.ctypes.data_as(_f64p), C.c_int64(b.shape[0]),
                                          C.c_int64(b.shape[1]), C.c_int64(sketch_rows),
                                          C.c_uint64(sketch_seed), _p(out)))
    return out


def select_order(taus, bound: float) -> int:
    t = f64(taus)
    return int(lib().orc_select_order(_p(t), C.c_int(t.size), C.c_double(bound)))


# ---------------------------------------------------------------- fits
class Fit(dict):
    __getattr__ = dict.__getitem__


def _unpack(packed, p_bar):
    out, off = [], 0
    for p in range(1, p_bar + 1):
        out.append(packed[off:off + p].copy())
        off += p
    return out


def lsar_fit(y, p_bar: int, c: int, seed: int, fixed_idx=None, fixed_w=None,
             want_scores_all: bool = False) -> Fit:
    y = f64(y)
    n = y.size
    w = max(n - p_bar, 1)
    pb = max(p_bar, 1)
    taus = np.zeros(pb); coefs = np.zeros(pb * (pb + 1) // 2); secs = np.zeros(pb)
    idx = np.zeros((pb, max(c, 1)), np.int64); wt = np.zeros((pb, max(c, 1)))
    rn = np.zeros(pb); ss = np.zeros(pb); sc = np.zeros(w); rr = np.zeros(w)
    meth = np.zeros(pb, np.int32)
    sall = np.zeros((pb, w)) if want_scores_all else None
    d = LsarDiag()
    if fixed_idx is not None:
        fixed_idx = i64(fixed_idx); fixed_w = f64(fixed_w)
        d.fixed_idx = _p(fixed_idx, _i64p); d.fixed_w = _p(fixed_w)
    d.idx_out = _p(idx, _i64p); d.w_out = _p(wt); d.rnorm2_out = _p(rn); d.ssum_out = _p(ss)
    d.scores_out = _p(sc); d.resid_out = _p(rr); d.method_out = _p(meth, _i32p)
    if sall is not None:
        d.scores_all = _p(sall)
    pstar = C.c_int(0)
    _check(lib().orc_lsar_fit(_p(y), C.c_int64(n), C.c_int(p_bar), C.c_int64(c), C.c_uint64(seed),
                              C.byref(d), _p(taus), _p(coefs), _p(secs), C.byref(pstar)))
    return Fit(taus=taus, coefs=_unpack(coefs, p_bar), lag_seconds=secs, p_star=pstar.value,
               idx=idx, w=wt, rnorm2=rn, ssum=ss, scores=sc, resid=rr, method=meth,
               scores_all=sall, bound=1.96 / np.sqrt(c))


def lsar_replay(y, p_bar: int, c: int, seed: int, coefs_packed) -> Fit:
    """orc_lsar_replay: the oracle's draws of a lsar_fit run from its coefficients."""
    y = f64(y); cf = f64(coefs_packed)
    if cf.size != p_bar * (p_bar + 1) // 2:
        raise OracleError(USAGE, "packed coefficients must hold p_bar (p_bar + 1) / 2 values")
    idx = np.zeros((p_bar, c), np.int64); w = np.zeros((p_bar, c)); rn = np.zeros(p_bar); ss = np.zeros(p_bar)
    _check(lib().orc_lsar_replay(_p(y), C.c_int64(y.size), C.c_int(p_bar), C.c_int64(c), C.c_uint64(seed),
                                 _p(cf), _p(idx, _i64p), _p(w), _p(rn), _p(ss)))
    return Fit(idx=idx, w=w, rnorm2=rn, ssum=ss)


def rh_replay(y, p_bar: int, c: int, seed: int, arow_idx, arow_w) -> Fit:
    """orc_rh_replay: final scores and per-lag draws from the final approximation rows."""
    y = f64(y); ai = i64(arow_idx); aw = f64(arow_w)
    m = y.size - p_bar
    scores = np.zeros(m); idx = np.zeros((p_bar, c), np.int64); w = np.zeros((p_bar, c))
    _check(lib().orc_rh_replay(_p(y), C.c_int64(y.size), C.c_int(p_bar), C.c_int64(c), C.c_uint64(seed),
                               _p(ai, _i64p), _p(aw), C.c_int64(ai.size), _p(scores), _p(idx, _i64p), _p(w)))
    return Fit(scores=scores, idx=idx, w=w)


def lsar_time_one_lag(y, p_bar: int, c: int, p: int, seed: int = 1) -> float:
    y = f64(y)
    return float(lib().orc_lsar_time_one_lag(_p(y), y.size, p_bar, c, p, seed))


def rh_time_upfront(y, p_bar: int, c: int, seed: int = 1) -> float:
    y = f64(y)
    return float(lib().orc_rh_time_upfront(_p(y), y.size, p_bar, c, seed))


def rh_defaults(m: int, k: int, c: int, seed: int) -> RhCfg:
    cfg = RhCfg()
    lib().orc_rh_defaults(C.c_int64(m), C.c_int64(k), C.c_int64(c), C.c_uint64(seed), C.byref(cfg))
    return cfg


def rh_fit(y, p_bar: int, c: int, seed: int, cfg: RhCfg | None = None, fixed_idx=None,
           fixed_w=None, want_levels: bool = False) -> Fit:
    y = f64(y)
    n = y.size
    m = max(n - p_bar, 1)
    k = p_bar + 1
    if cfg is None:
        ecfg = rh_defaults(m, k, c, derive_seed(seed, 0x5C07E5))
    else:
        ecfg = cfg
    pb = max(p_bar, 1)
    taus = np.zeros(pb); coefs = np.zeros(pb * (pb + 1) // 2); secs = np.zeros(pb)
    up = C.c_double(0); pstar = C.c_int(0); depth = C.c_int(0)
    scores = np.zeros(m)
    lsz = np.zeros(64, np.int64)
    sc = max(ecfg.sample_count, 1)
    maxdepth = 64
    upi = np.zeros((maxdepth, sc), np.int64); upw = np.zeros((maxdepth, sc))
    idx = np.zeros((pb, max(c, 1)), np.int64); wt = np.zeros((pb, max(c, 1)))
    arows_cap = max(ecfg.base_threshold, sc)
    approx = np.zeros(arows_cap * k)
    arows = C.c_int64(0)
    d = RhDiag()
    d.scores_out = _p(scores); d.depth_out = C.pointer(depth); d.level_sizes = _p(lsz, _i64p)
    lvl = None
    if want_levels:
        lvl = np.zeros(m, np.int64)
        d.level_idx = _p(lvl, _i64p); d.level_idx_cap = m
    d.up_idx = _p(upi, _i64p); d.up_w = _p(upw); d.idx_out = _p(idx, _i64p); d.w_out = _p(wt)
    d.approx_out = _p(approx); d.approx_rows = C.pointer(arows)
    if fixed_idx is not None:
        fixed_idx = i64(fixed_idx); fixed_w = f64(fixed_w)
        d.fixed_idx = _p(fixed_idx, _i64p); d.fixed_w = _p(fixed_w)
    _check(lib().orc_rh_fit(_p(y), C.c_int64(n), C.c_int(p_bar), C.c_int64(c),
                            C.byref(ecfg) if cfg is not None else None, C.c_uint64(seed),
                            C.byref(d), _p(taus), _p(coefs), _p(secs), C.byref(up),
                            C.byref(pstar)))
    dep = depth.value
    levels = None
    if want_levels:
        levels, off = [], 0
        for l in range(1, dep + 1):
            levels.append(lvl[off:off + lsz[l]].copy())
            off += lsz[l]
    ar = arows.value
    return Fit(taus=taus, coefs=_unpack(coefs, p_bar), lag_seconds=secs,
               upfront_seconds=up.value, p_star=pstar.value, scores=scores, depth=dep,
               level_sizes=lsz[:dep + 1].copy(), levels=levels, up_idx=upi[:dep].copy(),
               up_w=upw[:dep].copy(), idx=idx, w=wt,
               approx=approx[:ar * k].reshape(k, ar).T.copy(), cfg=ecfg,
               bound=1.96 / np.sqrt(c))


def exact_fit(y, p_bar: int) -> Fit:
    y = f64(y)
    taus = np.zeros(p_bar); coefs = np.zeros(p_bar * (p_bar + 1) // 2); pstar = C.c_int(0)
    _check(lib().orc_exact_fit(_p(y), C.c_int64(y.size), C.c_int(p_bar), _p(taus), _p(coefs),
                               C.byref(pstar)))
    return Fit(taus=taus, coefs=_unpack(coefs, p_bar), p_star=pstar.value,
               bound=1.96 / np.sqrt(y.size - p_bar))


# ---------------------------------------------------------------- SRHT (sketch.cpp:103-239)
def hadamard_apply(x) -> np.ndarray:
    v = f64(x).copy()
    _check(lib().orc_hadamard_apply(_p(v), C.c_int64(v.size)))
    return v


def srht_sample_count(n: int, d: int, epsilon: float):
    fv = C.c_double(0.0); c = C.c_int64(0); capped = C.c_int(0)
    _check(lib().orc_srht_sample_count(C.c_int64(n), C.c_int64(d), C.c_double(epsilon), C.byref(fv),
                                       C.byref(c), C.byref(capped)))
    return fv.value, c.value, bool(capped.value)


def srht_solve(a, b, c: int, seed: int):
    """a: rows x cols; returns (x, sampled a (c x cols), sampled b)."""
    a = np.asfortranarray(np.asarray(a, dtype=np.float64))
    b = f64(b)
    rows, cols = a.shape
    x = np.zeros(cols); sa = np.zeros((c, cols), order="F"); sb = np.zeros(c)
    _check(lib().orc_srht_solve(_p(a.ravel(order="F")), C.c_int64(rows), C.c_int64(cols), _p(b), C.c_int64(c),
                                C.c_uint64(seed), _p(x), _p(sa.ravel(order="F")), _p(sb)))
    return x, sa, sb


def srht_fit(y, p_bar: int, c: int, seed: int) -> Fit:
    y = f64(y)
    taus = np.zeros(max(p_bar, 1)); coefs = np.zeros(max(p_bar, 1) * (max(p_bar, 1) + 1) // 2)
    pstar = C.c_int(0)
    _check(lib().orc_srht_fit(_p(y), C.c_int64(y.size), C.c_int(p_bar), C.c_int64(c), C.c_uint64(seed),
                              _p(taus), _p(coefs), C.byref(pstar)))
    return Fit(taus=taus, coefs=_unpack(coefs, p_bar), p_star=pstar.value, bound=1.96 / np.sqrt(c))


# ---------------------------------------------------------------- generators
def random_stationary_ar(p: int, seed: int) -> np.ndarray:
    phi = np.empty(p)
    _check(lib().orc_random_stationary_ar(C.c_int(p), C.c_uint64(seed), _p(phi)))
    return phi


def simulate_ar(phi, n: int, seed: int, burn_in: int | None = None, noise_std: float = 1.0):
    phi = f64(phi)
    p = phi.size
    burn = 10 * p + 1000 if burn_in is None else burn_in
    out = np.empty(n)
    _check(lib().orc_simulate_ar(_p(phi), C.c_int(p), C.c_double(noise_std), C.c_int64(n),
                                 C.c_int64(burn), C.c_uint64(seed), _p(out)))
    return out
