"""Python mirror of the reference's fit API for the hot path.

Same names, argument meaning and error behaviour as namespace toepfit
(/root/reference/proj/include/toepfit):
  TimeSeries                       series.hpp:16-31
  UsageError/DataError/NumericalError   errors.hpp:12-29
  FitResult, PACFResult            lsar.hpp:28-35, toeplitz.hpp:59-66
  lsar_fit(series, p_bar, c, seed) lsar.hpp:89
  rh_fit(series, p_bar, c, config, seed)  repeated_halving.hpp:97-99
  RHConfig.defaults                repeated_halving.cpp:33-41
  run_fit(series, method, ...)     bench.cpp:107-124 (lsar | rh)
  report_to_json(report)           bench.cpp:268-283
  select_order(pacf)               toeplitz.cpp:133-138
Every call goes through the C ABI (libtoepfit_b200.so) onto the GPU.
"""
from __future__ import annotations

import ctypes as C
import json
import math
from dataclasses import dataclass, field

import numpy as np

from . import _abi
from ._abi import ptr


class UsageError(RuntimeError):
    pass


class DataError(RuntimeError):
    pass


class NumericalError(RuntimeError):
    pass


class CudaError(RuntimeError):
    pass


_ERRS = {_abi.TF_USAGE: UsageError, _abi.TF_DATA: DataError, _abi.TF_NUMERICAL: NumericalError,
         _abi.TF_CUDA: CudaError, _abi.TF_NCCL: CudaError}

EXIT_CODES = {UsageError: 2, DataError: 3, NumericalError: 4}  # errors.hpp:8-9


class TimeSeries:
    """Immutable fp64 series; validated non-empty and finite (series.cpp:23-32)."""

    def __init__(self, values, label: str = "", copy: bool = True):
        # copy=False keeps a read-only view of a contiguous fp64 array (e.g. a
        # pinned host buffer) instead of the owning copy the reference makes
        v = np.array(values, dtype=np.float64, copy=copy).ravel()
        if v.size == 0:
            raise DataError("series must contain at least one value")
        if not np.isfinite(v).all():
            raise DataError(f"series value at position {int(np.flatnonzero(~np.isfinite(v))[0])} is not finite")
        v.setflags(write=False)
        self._v = v
        self.label = label

    def values(self) -> np.ndarray:
        return self._v

    def size(self) -> int:
        return int(self._v.size)

    def __len__(self) -> int:
        return self.size()


def load_series_bin(path: str, *, pinned: bool = False) -> TimeSeries:
    """Read the reference's flat binary series (series.cpp:273-284, format
    series.hpp:93: uint64 little-endian count, then count f64 little-endian
    values), with its DataError messages.  pinned=True reads straight into
    page-locked host memory (a copy-free TimeSeries for a fast upload)."""
    try:
        f = open(path, "rb")
    except OSError:
        raise DataError("cannot open " + path) from None
    with f:
        head = f.read(8)
        if len(head) < 8:
            raise DataError(path + ": truncated header")
        count = int(np.frombuffer(head, dtype="<u8")[0])
        if pinned:
            import torch
            buf = torch.empty(count, dtype=torch.float64, pin_memory=True)
            arr = buf.numpy()
            got = f.readinto(memoryview(arr).cast("B")) if count else 0
            if got != 8 * count:
                raise DataError(path + ": truncated payload")
            ts = TimeSeries(arr, copy=False)
            ts._pinned = buf  # keep the page-locked buffer alive with the series
            return ts
        vals = np.fromfile(f, dtype="<f8", count=count)
        if vals.size != count:
            raise DataError(path + ": truncated payload")
    return TimeSeries(vals, copy=False)


def save_series_bin(series: TimeSeries, path: str) -> None:
    """Write the flat binary format (series.cpp:262-271)."""
    v = np.ascontiguousarray(series.values(), dtype="<f8")
    try:
        with open(path, "wb") as f:
            f.write(np.array([v.size], dtype="<u8").tobytes())
            v.tofile(f)
    except OSError:
        raise DataError("cannot write " + path) from None


@dataclass
class PACFResult:
    taus: list
    bound: float = 0.0
    method: str = "exact"


@dataclass
class FitResult:
    p_star: int = 0
    coefficients: np.ndarray = field(default_factory=lambda: np.zeros(0))
    pacf: PACFResult = field(default_factory=lambda: PACFResult([]))
    per_lag_seconds: list = field(default_factory=list)
    per_lag_coefficients: list = field(default_factory=list)
    upfront_seconds: float = 0.0
    diag: dict | None = None


@dataclass
class RHConfig:
    base_threshold: int = 0
    sample_count: int = 0
    gaussian_rows: int = 0
    seed: int = 0

    @staticmethod
    def defaults(n: int, k: int, c: int, seed: int) -> "RHConfig":
        logk = int(math.ceil(math.log(k + 1.0)))
        return RHConfig(base_threshold=max(c, 10 * k * logk), sample_count=c,
                        gaussian_rows=int(math.ceil(8.0 * math.log(max(n, 2)))), seed=seed)

    def validate(self) -> None:
        if self.sample_count < 1:
            raise UsageError("sample count must be positive")
        if self.base_threshold < self.sample_count:
            raise UsageError("base threshold below sample count")
        if self.gaussian_rows < 1:
            raise UsageError("need at least one sketch row")


def rh_level_sizes(m: int, base_threshold: int) -> list:
    """Halving level sizes m, m/2, ... while above the base (repeated_halving.cpp:130-145)."""
    sizes = [int(m)]
    while sizes[-1] > base_threshold:
        sizes.append(sizes[-1] // 2)
    return sizes


def derive_seed(seed: int, tag: int) -> int:
    return int(_abi.lib().tf_derive_seed(C.c_uint64(seed), C.c_uint64(tag)))


class Engine:
    """One tf_context (one CUDA device, one stream) with a resident series."""

    def __init__(self, device: int = 0, priority: int = 0):
        """priority: CUDA stream priority levels above the default (concurrent
        contexts on one GPU: the higher one's kernels are scheduled first)."""
        L = _abi.lib()
        self._ctx = C.c_void_p()
        opts = _abi.TfOpts(device=device, priority=int(priority))
        st = L.tf_create(C.byref(opts), C.byref(self._ctx))
        if st != _abi.TF_OK:
            raise CudaError(f"tf_create failed (status {st}); no usable CUDA device")
        self._series_id = None

    def close(self):
        if self._ctx:
            _abi.lib().tf_destroy(self._ctx)
            self._ctx = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, st: int):
        if st != _abi.TF_OK:
            msg = _abi.lib().tf_last_error(self._ctx).decode()
            raise _ERRS.get(st, RuntimeError)(msg)

    # ---------------------------------------------------------------- series
    def upload(self, series: TimeSeries):
        if self._series_id is not None and self._series_id[0] is series:
            return
        v = series.values()
        self._series_id = None  # a failed upload leaves no series resident
        self._check(_abi.lib().tf_upload_series(self._ctx, ptr(v), v.size))
        self._series_id = (series,)

    def forget_series(self):
        """Drop the resident-series cache: the next fit re-uploads (H2D) its series."""
        self._series_id = None

    def upload_device(self, dev_ptr: int, n: int):
        self._check(_abi.lib().tf_upload_series_device(self._ctx, C.c_void_p(dev_ptr), n))
        self._series_id = None

    # ---------------------------------------------------------------- sweeps
    def lsar_sweep_batch(self, ys, p_bar: int, c: int, seeds, fixed_idx=None, fixed_w=None, shared=False):
        """tf_lsar_sweep_batch: ys is a (B, n) array (or one series of n values
        with shared=True, fitted once per seed).  Returns taus (B, p_bar),
        packed coefficients (B, p_bar (p_bar+1)/2), per-lag batch seconds,
        p_star (B,) and status (B, 3)."""
        seeds = np.ascontiguousarray(np.asarray(seeds, dtype=np.uint64))
        B = int(seeds.size)
        y = np.ascontiguousarray(ys, dtype=np.float64)
        if shared:
            y = y.reshape(-1)
            n, stride = y.size, 0
        else:
            if y.ndim != 2 or y.shape[0] != B:
                raise UsageError("batch series must be a (len(seeds), n) array")
            n, stride = y.shape[1], y.shape[1]
        pb = max(int(p_bar), 1)
        taus = np.zeros((B, pb))
        coefs = np.zeros((B, pb * (pb + 1) // 2))
        secs = np.zeros(pb)
        pstar = np.zeros(B, np.int32)
        status = np.zeros((B, 3), np.int32)
        fi = fw = None
        if fixed_idx is not None:
            fi = np.ascontiguousarray(fixed_idx, dtype=np.int64)
            fw = np.ascontiguousarray(fixed_w, dtype=np.float64)
            if fi.size != B * pb * c or fw.size != B * pb * c:
                raise UsageError("fixed samples must be [batch][p_bar][c]")
        self._series_id = None  # a re-run fit replaces the resident series
        self._check(_abi.lib().tf_lsar_sweep_batch(
            self._ctx, ptr(y), int(stride), B, int(n), int(p_bar), int(c),
            seeds.ctypes.data_as(C.POINTER(C.c_uint64)),
            ptr(fi, _abi._i64p) if fi is not None else None, ptr(fw) if fw is not None else None,
            ptr(taus), ptr(coefs), ptr(secs), ptr(pstar, _abi._i32p), ptr(status, _abi._i32p)))
        return taus, coefs, secs, pstar, status

    def lsar_sweep(self, p_bar: int, c: int, seed: int, fixed_idx=None, fixed_w=None,
                   want_diag: bool = False, n: int | None = None, sharded: bool = False):
        """tf_lsar_sweep (or, sharded=True, tf_lsar_sweep_sharded on this rank's
        slice after tf_nccl_init -- see shard.NcclShard)."""
        pb = max(int(p_bar), 1)
        taus = np.zeros(pb)
        coefs = np.zeros(pb * (pb + 1) // 2)
        secs = np.zeros(pb)
        pstar = C.c_int(0)
        d = _abi.TfLsarDiag()
        keep = []
        diag = None
        if fixed_idx is not None:
            # fixed_w None: the weights of each lag's own distribution (k_fixed_weights)
            fi = np.ascontiguousarray(fixed_idx, dtype=np.int64)
            if fi.size != pb * c:
                raise UsageError("fixed samples must be [p_bar][c]")
            keep.append(fi)
            d.fixed_idx = ptr(fi, _abi._i64p)
            if fixed_w is not None:
                fw = np.ascontiguousarray(fixed_w, dtype=np.float64)
                if fw.size != pb * c:
                    raise UsageError("fixed samples must be [p_bar][c]")
                keep.append(fw)
                d.fixed_w = ptr(fw)
        if want_diag == "light":  # phases / methods / launches only (no per-row dumps)
            diag = dict(method=np.zeros(pb, np.int32), rank=np.zeros(pb, np.int32), phases=np.zeros((pb, 3)),
                        launches=np.zeros(1, np.int64), svd_sweeps=np.zeros(pb, np.int32))
            d.method_out = ptr(diag["method"], _abi._i32p)
            d.rank_out = ptr(diag["rank"], _abi._i32p)
            d.svd_sweeps_out = ptr(diag["svd_sweeps"], _abi._i32p)
            d.phase_seconds = ptr(diag["phases"])
            d.launches_out = ptr(diag["launches"], _abi._i64p)
        elif want_diag:
            w = max(int(n) - pb, 1)
            diag = dict(idx=np.zeros((pb, c), np.int64), w=np.zeros((pb, c)), rnorm2=np.zeros(pb),
                        ssum=np.zeros(pb), scores=np.zeros(w), resid=np.zeros(w),
                        method=np.zeros(pb, np.int32), rank=np.zeros(pb, np.int32), phases=np.zeros((pb, 3)),
                        launches=np.zeros(1, np.int64))
            d.rank_out = ptr(diag["rank"], _abi._i32p)
            d.idx_out = ptr(diag["idx"], _abi._i64p)
            d.w_out = ptr(diag["w"])
            d.rnorm2_out = ptr(diag["rnorm2"])
            d.ssum_out = ptr(diag["ssum"])
            d.scores_out = ptr(diag["scores"])
            d.resid_out = ptr(diag["resid"])
            d.method_out = ptr(diag["method"], _abi._i32p)
            d.phase_seconds = ptr(diag["phases"])
            d.launches_out = ptr(diag["launches"], _abi._i64p)
        fn = _abi.lib().tf_lsar_sweep_sharded if sharded else _abi.lib().tf_lsar_sweep
        self._check(fn(self._ctx, int(p_bar), int(c), C.c_uint64(seed), C.byref(d), ptr(taus), ptr(coefs), ptr(secs),
                       C.byref(pstar)))
        return taus, coefs, secs, pstar.value, diag

    def rh_sweep(self, p_bar: int, c: int, cfg: RHConfig | None, seed: int, fixed=None,
                 want_diag: bool = False, n: int | None = None):
        pb = max(int(p_bar), 1)
        taus = np.zeros(pb)
        coefs = np.zeros(pb * (pb + 1) // 2)
        secs = np.zeros(pb)
        up = C.c_double(0)
        pstar = C.c_int(0)
        d = _abi.TfRhDiag()
        keep = []
        diag = None
        if fixed:
            for key, attr, dt in (("idx", "fixed_idx", np.int64), ("w", "fixed_w", np.float64),
                                  ("levels", "fixed_levels", np.int64),
                                  ("up_idx", "fixed_up_idx", np.int64),
                                  ("up_w", "fixed_up_w", np.float64)):
                if fixed.get(key) is not None:
                    a = np.ascontiguousarray(fixed[key], dtype=dt).ravel()
                    keep.append(a)
                    setattr(d, attr, ptr(a, _abi._i64p if dt == np.int64 else _abi._f64p))
        depth = C.c_int(0)
        if want_diag:
            m = max(int(n) - pb, 1)
            ecfg = cfg if cfg is not None else RHConfig.defaults(m, pb + 1, c, derive_seed(seed, 0x5C07E5))
            sizes = rh_level_sizes(m, ecfg.base_threshold)
            sc = max(int(ecfg.sample_count), 1)
            dep = len(sizes) - 1
            diag = dict(scores=np.zeros(m), idx=np.zeros((pb, c), np.int64), w=np.zeros((pb, c)),
                        levels_flat=np.zeros(max(sum(sizes[1:]), 1), np.int64),
                        up_idx=np.zeros((max(dep, 1), sc), np.int64), up_w=np.zeros((max(dep, 1), sc)),
                        level_sizes=sizes)
            d.scores_out = ptr(diag["scores"])
            d.idx_out = ptr(diag["idx"], _abi._i64p)
            d.w_out = ptr(diag["w"])
            d.depth_out = C.pointer(depth)
            d.levels_out = ptr(diag["levels_flat"], _abi._i64p)
            d.up_idx_out = ptr(diag["up_idx"], _abi._i64p)
            d.up_w_out = ptr(diag["up_w"])
            diag["launches"] = np.zeros(1, np.int64)
            d.launches_out = ptr(diag["launches"], _abi._i64p)
            diag["method"] = np.zeros(pb, np.int32)
            diag["rank"] = np.zeros(pb, np.int32)
            d.method_out = ptr(diag["method"], _abi._i32p)
            d.rank_out = ptr(diag["rank"], _abi._i32p)
        ccfg = None
        if cfg is not None:
            ccfg = _abi.TfRhCfg(cfg.base_threshold, cfg.sample_count, cfg.gaussian_rows, cfg.seed)
        self._check(_abi.lib().tf_rh_sweep(self._ctx, int(p_bar), int(c),
                                           C.byref(ccfg) if ccfg is not None else None,
                                           C.c_uint64(seed), C.byref(d), ptr(taus), ptr(coefs),
                                           ptr(secs), C.byref(up), C.byref(pstar)))
        if diag is not None:
            diag["depth"] = depth.value
            sizes, off, levels = diag["level_sizes"], 0, []
            for l in range(1, len(sizes)):
                levels.append(diag["levels_flat"][off:off + sizes[l]])
                off += sizes[l]
            diag["levels"] = levels
            diag["up_idx"] = diag["up_idx"][:depth.value]
            diag["up_w"] = diag["up_w"][:depth.value]
        return taus, coefs, secs, up.value, pstar.value, diag

    def generate_series(self, roots, n: int, seed: int, innovations: str = "normal", burn_in: int = 1000):
        """Synthetic AR series generated on the device and kept resident (the
        sweeps then run on it without a host copy)."""
        r = np.ascontiguousarray(roots, dtype=np.float64)
        self._check(_abi.lib().tf_generate_series(self._ctx, ptr(r), int(r.size), int(n), C.c_uint64(seed),
                                                  1 if innovations == "t3" else 0, int(burn_in)))
        self._series_id = ("device", int(n))
        return int(n)

    def download_series(self, n: int) -> np.ndarray:
        out = np.empty(int(n))
        self._check(_abi.lib().tf_download_series(self._ctx, ptr(out), int(n)))
        return out

    def download_series_into(self, out: np.ndarray) -> None:
        """D2H of the resident series into a caller buffer (e.g. pinned host memory)."""
        if out.dtype != np.float64 or not out.flags.c_contiguous:
            raise UsageError("output must be a contiguous float64 array")
        self._check(_abi.lib().tf_download_series(self._ctx, ptr(out), int(out.size)))

    def exact_sweep(self, p_bar: int):
        pb = max(int(p_bar), 1)
        taus = np.zeros(pb)
        coefs = np.zeros(pb * (pb + 1) // 2)
        secs = np.zeros(pb)
        pstar = C.c_int(0)
        self._check(_abi.lib().tf_exact_sweep(self._ctx, int(p_bar), ptr(taus), ptr(coefs), ptr(secs),
                                              C.byref(pstar)))
        return taus, coefs, secs, pstar.value

    def srht_sweep(self, p_bar: int, c: int, seed: int):
        pb = max(int(p_bar), 1)
        taus = np.zeros(pb)
        coefs = np.zeros(pb * (pb + 1) // 2)
        secs = np.zeros(pb)
        pstar = C.c_int(0)
        self._check(_abi.lib().tf_srht_sweep(self._ctx, int(p_bar), int(c), int(seed) & (2**64 - 1), ptr(taus),
                                             ptr(coefs), ptr(secs), C.byref(pstar)))
        return taus, coefs, secs, pstar.value

    def hadamard(self, x) -> np.ndarray:
        v = np.array(x, dtype=np.float64).ravel()
        self._check(_abi.lib().tf_hadamard(self._ctx, ptr(v), v.size))
        return v

    def sweep_span(self, ref: "Engine"):
        """(start_ms, end_ms) of this engine's last sweep relative to the start
        of ref's last sweep (device events)."""
        a, b = C.c_double(0), C.c_double(0)
        self._check(_abi.lib().tf_sweep_span(ref._ctx, self._ctx, C.byref(a), C.byref(b)))
        return a.value, b.value

    def probe_fp64_peak(self) -> float:
        v = C.c_double(0)
        self._check(_abi.lib().tf_probe_fp64_peak(self._ctx, C.byref(v)))
        return v.value

    def fft_first_lag(self, p_bar: int) -> int:
        """First lag of a p_bar sweep whose pass runs the FFT FIR (p_bar + 1: none)."""
        v = C.c_int(0)
        self._check(_abi.lib().tf_fft_first_lag(self._ctx, int(p_bar), C.byref(v)))
        return v.value

    # ------------------------------------------------------------ single ops
    def residuals(self, y, n_used: int, p: int, phi) -> np.ndarray:
        y = np.ascontiguousarray(y, dtype=np.float64)
        phi = np.ascontiguousarray(phi, dtype=np.float64)
        if phi.size != p:
            raise UsageError("coefficient length does not match lag order")
        out = np.zeros(max(n_used - p, 1))
        self._check(_abi.lib().tf_residuals(self._ctx, ptr(y), int(n_used), int(p), ptr(phi), ptr(out)))
        self._series_id = None
        return out[: n_used - p]

    def sample_rows(self, scores, c: int, seed: int):
        s = np.ascontiguousarray(scores, dtype=np.float64)
        idx = np.zeros(max(c, 1), np.int64)
        w = np.zeros(max(c, 1))
        self._check(_abi.lib().tf_sample_rows(self._ctx, ptr(s), s.size, int(c), C.c_uint64(seed),
                                              ptr(idx, _abi._i64p), ptr(w)))
        return idx[:c], w[:c]

    def apply_sample(self, y, n_used: int, p: int, idx, w, width: int | None = None):
        y = np.ascontiguousarray(y, dtype=np.float64)
        idx = np.ascontiguousarray(idx, dtype=np.int64)
        w = np.ascontiguousarray(w, dtype=np.float64)
        width = p if width is None else width
        a = np.zeros((idx.size, max(width, 1)))
        b = np.zeros(idx.size)
        self._check(_abi.lib().tf_apply_sample(self._ctx, ptr(y), int(n_used), int(p),
                                               ptr(idx, _abi._i64p), ptr(w), idx.size, int(width),
                                               ptr(a), ptr(b)))
        self._series_id = None
        return a, b

    def solve_sampled(self, y, n_used: int, p: int, idx, w):
        y = np.ascontiguousarray(y, dtype=np.float64)
        idx = np.ascontiguousarray(idx, dtype=np.int64)
        w = np.ascontiguousarray(w, dtype=np.float64)
        phi = np.zeros(p)
        m = C.c_int(0)
        self._check(_abi.lib().tf_solve_sampled(self._ctx, ptr(y), int(n_used), int(p),
                                                ptr(idx, _abi._i64p), ptr(w), idx.size, ptr(phi),
                                                C.byref(m)))
        self._series_id = None
        return phi, m.value


_default_engine: Engine | None = None


def default_engine() -> Engine:
    global _default_engine
    if _default_engine is None:
        _default_engine = Engine(0)
    return _default_engine


def _unpack(coefs, p_bar):
    out, off = [], 0
    for p in range(1, p_bar + 1):
        out.append(coefs[off:off + p].copy())
        off += p
    return out


def _finish(method, taus, coefs, secs, pstar, p_bar, c, upfront=0.0, diag=None) -> FitResult:
    per = _unpack(coefs, p_bar)
    fit = FitResult()
    fit.pacf = PACFResult(taus=list(map(float, taus)), bound=1.96 / math.sqrt(float(c)), method=method)
    fit.per_lag_seconds = list(map(float, secs))
    fit.per_lag_coefficients = per
    fit.p_star = int(pstar)
    fit.coefficients = per[pstar - 1].copy() if pstar > 0 else np.zeros(0)
    fit.upfront_seconds = float(upfront)
    fit.diag = diag
    return fit


@dataclass
class LeverageState:
    """lsar.hpp:17-23: the recursion's state after the compressed solve at lag p."""
    p: int = 0
    m: int = 0
    scores: np.ndarray = field(default_factory=lambda: np.zeros(0))
    residuals: np.ndarray = field(default_factory=lambda: np.zeros(0))
    coefficients: np.ndarray = field(default_factory=lambda: np.zeros(0))
    method: int = 0


class LsarDriver:
    """lsar.hpp:65-84 (LsarDriver): the LSAR recursion one lag at a time on the
    GPU (tf_lsar_step).  first_lag() / advance(state) return host states like
    the reference; advance() of the state the previous call returned continues
    from the device-resident vectors (no upload), any other state is uploaded."""

    def __init__(self, series: TimeSeries, p_bar: int, c: int, seed: int, *, engine: Engine | None = None):
        if p_bar < 1:
            raise UsageError("maximum lag must be at least 1")
        if series.size() <= p_bar + 1:
            raise DataError(f"series too short for maximum lag {p_bar}")
        if c < p_bar:
            raise UsageError("sample count below maximum lag")
        self.series, self.p_bar, self.c, self.seed = series, int(p_bar), int(c), int(seed)
        self.eng = engine or default_engine()
        self._w = series.size() - p_bar
        self._last = None

    def row_count(self) -> int:
        return self._w

    def window_length(self, p: int) -> int:
        """window_system(p) covers the first n - p_bar + p observations (lsar.cpp:66-68)."""
        return self._w + p

    def _step(self, p: int, prev: LeverageState | None) -> LeverageState:
        self.eng.upload(self.series)
        w = self._w
        sc, rs, phi, m = np.zeros(w), np.zeros(w), np.zeros(p), C.c_int(0)
        resident = prev is not None and prev is self._last
        s_in = r_in = None
        if prev is not None and not resident:
            s_in = np.ascontiguousarray(prev.scores, dtype=np.float64)
            r_in = np.ascontiguousarray(prev.residuals, dtype=np.float64)
            if s_in.size != w or r_in.size != w:
                raise UsageError("state vectors must hold row_count() values")
        self.eng._check(_abi.lib().tf_lsar_step(self.eng._ctx, self.p_bar, self.c, C.c_uint64(self.seed), int(p),
                                                ptr(s_in), ptr(r_in), ptr(sc), ptr(rs), ptr(phi), C.byref(m)))
        st = LeverageState(p=p, m=w + p, scores=sc, residuals=rs, coefficients=phi, method=m.value)
        self._last = st
        return st

    def first_lag(self) -> LeverageState:
        return self._step(1, None)

    def advance(self, state: LeverageState) -> LeverageState:
        if state.p < 1 or state.p >= self.p_bar:
            raise UsageError("cannot advance past maximum lag")  # lsar.cpp:90
        return self._step(state.p + 1, state)


# ---------------------------------------------------------------- RowSource / RH over a row source
@dataclass
class GaussianSketch:
    """sketch.hpp GaussianSketch: `rows` Gaussian mixes drawn from Rng(seed)."""
    rows: int
    seed: int


class RowSource:
    """repeated_halving.hpp:17-23: read-only row access to an n x k matrix that may
    never exist in memory.  Subclasses implement rows(), cols(), gather(idx)."""

    def rows(self) -> int:
        raise NotImplementedError

    def cols(self) -> int:
        raise NotImplementedError

    def gather(self, idx: np.ndarray) -> np.ndarray:
        raise NotImplementedError


class DenseRowSource(RowSource):
    def __init__(self, a):
        self.a = np.ascontiguousarray(np.asarray(a, dtype=np.float64))

    def rows(self) -> int:
        return int(self.a.shape[0])

    def cols(self) -> int:
        return int(self.a.shape[1])

    def gather(self, idx):
        return self.a[np.asarray(idx, dtype=np.int64)]


class AugmentedRowSource(RowSource):
    """Rows of the augmented lag-p system [T, b] (repeated_halving.cpp:22-31):
    row i = (y[p+i-1], ..., y[i], y[p+i]) over the first n_used observations."""

    def __init__(self, series: TimeSeries, p: int, n_used: int | None = None):
        self.y = series.values()
        self.p = int(p)
        self.n_used = int(n_used) if n_used is not None else series.size()
        if self.p < 1:
            raise UsageError("lag order must be at least 1")
        if self.n_used <= self.p:
            raise DataError("series window too short for lag order")

    def rows(self) -> int:
        return self.n_used - self.p

    def cols(self) -> int:
        return self.p + 1

    def gather(self, idx):
        i = np.asarray(idx, dtype=np.int64)[:, None]
        cols = np.concatenate([self.p - 1 - np.arange(self.p), [self.p]])
        return self.y[i + cols[None, :]]


@dataclass
class SpectralApprox:
    """repeated_halving.hpp:49-53."""
    rows: np.ndarray
    levels: int = 0
    sample_count: int = 0


def generalized_leverage(c_rows, b, sketch: GaussianSketch | None = None, *, engine: Engine | None = None):
    """repeated_halving.hpp:76-78 on the GPU (tf_generalized_leverage)."""
    eng = engine or default_engine()
    c_rows = np.ascontiguousarray(np.asarray(c_rows, dtype=np.float64))
    b = np.ascontiguousarray(np.asarray(b, dtype=np.float64))
    if c_rows.ndim != 2 or b.ndim != 2:
        raise UsageError("matrices must be 2-D")
    out = np.zeros(max(c_rows.shape[0], 1))
    g, sd = (int(sketch.rows), int(sketch.seed)) if sketch is not None else (0, 0)
    eng._check(_abi.lib().tf_generalized_leverage(eng._ctx, ptr(c_rows), c_rows.shape[0], c_rows.shape[1], ptr(b),
                                                  b.shape[0], b.shape[1], g, C.c_uint64(sd), ptr(out)))
    return out[:c_rows.shape[0]]


def repeated_halving(x: RowSource, config: RHConfig, *, engine: Engine | None = None) -> SpectralApprox:
    """repeated_halving.hpp:83-86 on the GPU over a host row source (tf_repeated_halving)."""
    config.validate()
    eng = engine or default_engine()
    n, k = int(x.rows()), int(x.cols())
    errors = []

    def _gather(user, idx, count, out):
        try:
            ids = np.ctypeslib.as_array(idx, shape=(count,)).copy() if count else np.zeros(0, np.int64)
            rows = np.ascontiguousarray(np.asarray(x.gather(ids), dtype=np.float64)).reshape(count, k)
            if count:
                np.ctypeslib.as_array(out, shape=(count * k,))[:] = rows.ravel()
        except Exception as e:  # never unwind through the C ABI
            errors.append(e)

    cb = _abi.GATHER_FN(_gather)
    cap = max(config.sample_count, config.base_threshold, n if n <= config.base_threshold else 0, 1)
    approx = np.zeros((cap, k))
    arows = C.c_int64(0)
    lev = C.c_int(0)
    cfg = _abi.TfRhCfg(config.base_threshold, config.sample_count, config.gaussian_rows, config.seed)
    st = _abi.lib().tf_repeated_halving(eng._ctx, n, k, cb, None, C.byref(cfg), ptr(approx), cap, C.byref(arows),
                                        C.byref(lev))
    if errors:
        raise errors[0]
    eng._check(st)
    return SpectralApprox(rows=approx[:arows.value].copy(), levels=lev.value, sample_count=int(arows.value))


def rh_leverage_scores(series: TimeSeries, p: int, config: RHConfig, *, engine: Engine | None = None):
    """repeated_halving.hpp:88-91: scores of every row of the augmented lag-p
    system against its RH approximation (final pass unsketched)."""
    src = AugmentedRowSource(series, p)
    approx = repeated_halving(src, config, engine=engine)
    return generalized_leverage(src.gather(np.arange(src.rows())), approx.rows, None, engine=engine)


def lsar_fit(series: TimeSeries, p_bar: int, c: int, seed: int, *, engine: Engine | None = None,
             fixed_idx=None, fixed_w=None, want_diag: bool = False) -> FitResult:
    """lsar.cpp:100-124 on the GPU.  fixed_idx/fixed_w ([p_bar][c]) switch to
    deterministic-index mode (samples supplied instead of drawn)."""
    eng = engine or default_engine()
    eng.upload(series)
    taus, coefs, secs, pstar, diag = eng.lsar_sweep(p_bar, c, seed, fixed_idx, fixed_w, want_diag,
                                                    n=series.size())
    return _finish("lsar", taus, coefs, secs, pstar, p_bar, c, 0.0, diag)


_BATCH_REASONS = {1: "zero residual norm; sampling distribution undefined", 2: "negative leverage score",
                  3: "zero score sum; distribution undefined", 4: "compressed least-squares factorization failed",
                  6: "all-zero window; leverage undefined"}
_BATCH_ERRS = {1: UsageError, 2: DataError, 3: NumericalError}


def lsar_fit_batch(series_list, p_bar: int, c: int, seeds, *, engine: Engine | None = None,
                   fixed_idx=None, fixed_w=None, errors: str = "raise") -> list:
    """Many independent LSAR fits in one batched sweep (tf_lsar_sweep_batch):
    fit b = lsar_fit(series_list[b], p_bar, c, seeds[b]) (lsar.cpp:100-124).
    series_list: equal-length series (a list or a (B, n) array), or a single
    TimeSeries / 1-D array fitted once per seed (the reference's multi-seed
    run_compare / run_sweep loops, bench.cpp:183-188, 221-228).  p_bar <= 63.
    per_lag_seconds are the batch's per-lag device times divided by the
    number of fits (the amortised cost of one fit).  errors="raise"
    raises the first failing fit's UsageError / DataError / NumericalError;
    "return" puts the exception in that fit's slot instead."""
    eng = engine or default_engine()
    seeds = list(seeds)
    if isinstance(series_list, TimeSeries) or (isinstance(series_list, np.ndarray) and series_list.ndim == 1):
        y = series_list.values() if isinstance(series_list, TimeSeries) else series_list
        out = eng.lsar_sweep_batch(y, p_bar, c, seeds, fixed_idx, fixed_w, shared=True)
    elif isinstance(series_list, np.ndarray):  # (B, n): used in place
        out = eng.lsar_sweep_batch(series_list, p_bar, c, seeds, fixed_idx, fixed_w)
    else:
        rows = [s.values() if isinstance(s, TimeSeries) else np.asarray(s, dtype=np.float64) for s in series_list]
        if len({r.size for r in rows}) > 1:
            raise UsageError("batched fits need equal-length series")
        out = eng.lsar_sweep_batch(np.stack(rows) if rows else np.zeros((0, 0)), p_bar, c, seeds, fixed_idx,
                                   fixed_w)
    taus, coefs, secs, pstar, status = out
    fits = []
    for b in range(len(seeds)):
        code, lag, reason = (int(v) for v in status[b])
        if code:
            err = _BATCH_ERRS.get(code, NumericalError)(
                f"fit {b}: {_BATCH_REASONS.get(reason, 'numerical failure')} (lag {lag})")
            if errors == "raise":
                raise err
            fits.append(err)
            continue
        fits.append(_finish("lsar", taus[b], coefs[b], secs / len(seeds), int(pstar[b]), p_bar, c))
    return fits


def _lsar_reps(series: TimeSeries, p_bar: int, c: int, seeds, workers: int) -> list:
    """The LSAR repetitions of run_compare / run_sweep (many seeds over one
    series): one batched sweep sharing the series (tf_lsar_sweep_batch,
    y_stride 0) where the batch supports p_bar, else concurrent single fits."""
    if 1 <= p_bar <= 63:
        return lsar_fit_batch(series, p_bar, c, seeds)
    return fit_many([series] * len(seeds), "lsar", p_bar, c, seeds, workers=workers)


def rh_fit(series: TimeSeries, p_bar: int, c: int, config: RHConfig | None = None, seed: int = 0, *,
           engine: Engine | None = None, fixed=None, want_diag: bool = False) -> FitResult:
    """repeated_halving.cpp:191-232 on the GPU."""
    eng = engine or default_engine()
    eng.upload(series)
    taus, coefs, secs, up, pstar, diag = eng.rh_sweep(p_bar, c, config, seed, fixed, want_diag,
                                                      n=series.size())
    return _finish("rh", taus, coefs, secs, pstar, p_bar, c, up, diag)


def exact_fit(series: TimeSeries, p_bar: int, *, engine: Engine | None = None) -> FitResult:
    """Exact per-lag OLS on the full series (bench.cpp:27-48) on the GPU."""
    eng = engine or default_engine()
    eng.upload(series)
    taus, coefs, secs, pstar = eng.exact_sweep(p_bar)
    fit = _finish("exact", taus, coefs, secs, pstar, p_bar, 1, 0.0, None)
    fit.pacf.bound = 1.96 / math.sqrt(float(series.size() - p_bar))
    return fit


def srht_fit(series: TimeSeries, p_bar: int, c: int, seed: int, *, engine: Engine | None = None) -> FitResult:
    """Subsampled randomized Hadamard transform fit (bench.cpp:50-72): lag h
    solves the SRHT sketch (sketch.cpp:187-239, seed derive_seed(seed, h)) of
    its n - h row system on the GPU."""
    eng = engine or default_engine()
    eng.upload(series)
    taus, coefs, secs, pstar = eng.srht_sweep(p_bar, c, seed)
    fit = _finish("srht", taus, coefs, secs, pstar, p_bar, c, 0.0, None)
    fit.pacf.bound = 1.96 / math.sqrt(float(c))
    return fit


def hadamard_apply(x, *, engine: Engine | None = None) -> np.ndarray:
    """Orthonormal Walsh-Hadamard transform (sketch.cpp:107-120) on the GPU;
    UsageError unless the length is a power of two."""
    return (engine or default_engine()).hadamard(x)


@dataclass
class SrhtCount:
    c: int
    formula_value: float
    capped: bool


def srht_sample_count(n: int, d: int, epsilon: float) -> SrhtCount:
    """sketch.cpp:165-185 (host arithmetic)."""
    if not (n > d >= 1):
        raise UsageError("need n > d >= 1")
    if not (0.0 < epsilon < 1.0):
        raise UsageError("epsilon must lie in (0, 1)")
    nd = float(n) * float(d)
    log_term = math.log(40.0 * nd)
    branch1 = 48.0 * 48.0 * float(d) * log_term * math.log(100.0 * 100.0 * d * log_term)
    branch2 = 40.0 * float(d) * log_term / epsilon
    fv = max(branch1, branch2)
    rounded = math.ceil(fv)
    if rounded > n:
        return SrhtCount(int(n), fv, True)
    return SrhtCount(int(rounded), fv, False)


def fit_many(series_list, method: str, p_bar: int, c: int, seeds, *, workers: int = 8,
             device: int = 0, config: RHConfig | None = None) -> list:
    """Independent fits (many series, or many seeds over one series -- the
    reference's run_compare / run_sweep loops, bench.cpp:183-188, 221-228, and
    the BASELINE C5 batch) run concurrently: `workers` contexts, one CUDA
    stream each, fed from a shared queue (independent fits may run
    concurrently).  Returns FitResults in input order."""
    import threading
    items = list(zip(series_list, seeds))
    out = [None] * len(items)
    errors = []
    lock = threading.Lock()
    nxt = [0]

    def work():
        eng = Engine(device)
        try:
            while True:
                with lock:
                    k = nxt[0]
                    nxt[0] += 1
                if k >= len(items) or errors:
                    return
                ser, seed = items[k]
                if not isinstance(ser, TimeSeries):
                    ser = TimeSeries(ser)
                if method == "lsar":
                    out[k] = lsar_fit(ser, p_bar, c, seed, engine=eng)
                elif method == "rh":
                    out[k] = rh_fit(ser, p_bar, c, config, seed, engine=eng)
                elif method == "exact":
                    out[k] = exact_fit(ser, p_bar, engine=eng)
                elif method == "srht":
                    out[k] = srht_fit(ser, p_bar, c, seed, engine=eng)
                else:
                    raise UsageError(f"unknown method '{method}'")
        except Exception as e:  # noqa: BLE001 -- re-raised in the caller
            errors.append(e)
        finally:
            eng.close()

    th = [threading.Thread(target=work) for _ in range(max(1, min(workers, len(items))))]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if errors:
        raise errors[0]
    return out


def select_order(pacf: PACFResult) -> int:
    t = np.ascontiguousarray(pacf.taus, dtype=np.float64)
    return int(_abi.lib().tf_select_order(ptr(t), t.size, float(pacf.bound)))


@dataclass
class RunReport:
    method: str
    n: int
    p_bar: int
    c: int
    seed: int
    timing_recorded: bool
    upfront_seconds: float
    per_lag_seconds: list
    cumulative_seconds: list
    pacf: PACFResult
    p_star: int
    coefficients: list


def run_fit(series: TimeSeries, method: str, p_bar: int, c: int, seed: int,
            with_timing: bool = True, engine: Engine | None = None) -> RunReport:
    """bench.cpp:107-124: exact | lsar | rh | srht, all on the GPU."""
    if method != "exact" and c < 1:
        raise UsageError(f"method '{method}' needs a sample count")
    if method == "exact":
        fit = exact_fit(series, p_bar, engine=engine)
    elif method == "lsar":
        fit = lsar_fit(series, p_bar, c, seed, engine=engine)
    elif method == "rh":
        fit = rh_fit(series, p_bar, c, None, seed, engine=engine)
    elif method == "srht":
        fit = srht_fit(series, p_bar, c, seed, engine=engine)
    else:
        raise UsageError(f"unknown method '{method}'")
    if not with_timing:  # bench.cpp:76-79
        fit.per_lag_seconds = [0.0] * len(fit.per_lag_seconds)
        fit.upfront_seconds = 0.0
    cum, acc = [], fit.upfront_seconds
    for s in fit.per_lag_seconds:
        acc += s
        cum.append(acc)
    return RunReport(method=method, n=series.size(), p_bar=p_bar, c=c, seed=seed,
                     timing_recorded=with_timing, upfront_seconds=fit.upfront_seconds,
                     per_lag_seconds=fit.per_lag_seconds, cumulative_seconds=cum, pacf=fit.pacf,
                     p_star=fit.p_star, coefficients=list(map(float, fit.coefficients)))


def report_to_json(r: RunReport) -> str:
    """bench.cpp:268-283 key order and layout (nlohmann dump(2))."""
    j = {"method": r.method, "n": r.n, "p_bar": r.p_bar, "c": r.c, "seed": r.seed,
         "timing_recorded": r.timing_recorded, "upfront_seconds": r.upfront_seconds,
         "per_lag_seconds": r.per_lag_seconds, "cumulative_seconds": r.cumulative_seconds,
         "pacf": {"method": r.pacf.method, "bound": r.pacf.bound, "taus": r.pacf.taus},
         "p_star": r.p_star, "coefficients": r.coefficients}
    return json.dumps(j, indent=2, sort_keys=True) + "\n"  # nlohmann objects are key-sorted


# ---------------------------------------------------------------------------
# Comparison drivers (bench.cpp:126-243): the callers that run many seeds of
# lsar / rh against one exact fit.  The repetitions are independent fits and
# run concurrently on the device (fit_many: one context and stream each).
def relative_error_pct(estimate, reference) -> float:
    """toeplitz.cpp:140-146."""
    e = np.asarray(estimate, dtype=np.float64)
    r = np.asarray(reference, dtype=np.float64)
    if e.size != r.size:
        raise UsageError("length mismatch")
    ref_norm = float(np.linalg.norm(r))
    if ref_norm == 0.0:
        raise NumericalError("reference coefficients have zero norm")
    return 100.0 * float(np.linalg.norm(e - r)) / ref_norm


def trimmed_mean(values, trim_fraction: float) -> float:
    """bench.cpp:126-139."""
    v = sorted(float(x) for x in values)
    if not v:
        raise UsageError("trimmed mean of an empty sample")
    if not (0.0 <= trim_fraction < 0.5):
        raise UsageError("trim fraction must lie in [0, 0.5)")
    drop = int(math.floor(trim_fraction * len(v)))
    kept = v[drop:len(v) - drop]
    acc = 0.0
    for x in kept:  # sequential, as std::accumulate
        acc += x
    return acc / len(kept)


@dataclass
class MethodComparison:
    method: str
    trimmed_error_pct: list
    mean_lag_seconds: list
    mean_upfront_seconds: float
    p_stars: list


@dataclass
class CompareReport:
    n: int
    p_bar: int
    c: int
    repetitions: int
    trim_fraction: float
    seed: int
    timing_recorded: bool
    exact_p_star: int
    exact_lag_seconds: list
    exact_taus: list
    lsar: MethodComparison
    rh: MethodComparison


@dataclass
class SweepRow:
    method: str
    c: int
    max_lag_seconds: float
    max_error_pct: float


def _strip_timing(f: FitResult) -> None:
    f.per_lag_seconds = [0.0] * len(f.per_lag_seconds)
    f.upfront_seconds = 0.0


def _summarize(method: str, exact: FitResult, runs: list, trim_fraction: float) -> MethodComparison:
    """bench.cpp:143-168."""
    p_bar = len(exact.per_lag_coefficients)
    reps = len(runs)
    err, secs = [], []
    for h in range(p_bar):
        errs = [relative_error_pct(r.per_lag_coefficients[h], exact.per_lag_coefficients[h]) for r in runs]
        acc = 0.0
        for r in runs:
            acc += r.per_lag_seconds[h]
        secs.append(acc / reps)
        err.append(trimmed_mean(errs, trim_fraction))
    up = 0.0
    for r in runs:
        up += r.upfront_seconds
    return MethodComparison(method, err, secs, up / reps, [r.p_star for r in runs])


def run_compare(series: TimeSeries, p_bar: int, c: int, reps: int, trim_fraction: float, seed: int,
                with_timing: bool = True, *, workers: int = 8) -> CompareReport:
    """bench.cpp:172-212: one exact fit, `reps` LSAR and RH fits with seeds
    derive_seed(seed, 0x1000 + r) / derive_seed(seed, 0x2000 + r)."""
    if reps < 1:
        raise UsageError("need at least one repetition")
    if not (0.0 <= trim_fraction < 0.5):
        raise UsageError("trim fraction must lie in [0, 0.5)")
    exact = exact_fit(series, p_bar)
    lsar_runs = _lsar_reps(series, p_bar, c, [derive_seed(seed, 0x1000 + r) for r in range(reps)], workers)
    rh_runs = fit_many([series] * reps, "rh", p_bar, c, [derive_seed(seed, 0x2000 + r) for r in range(reps)],
                       workers=workers)
    if not with_timing:
        for f in [exact] + lsar_runs + rh_runs:
            _strip_timing(f)
    return CompareReport(n=series.size(), p_bar=p_bar, c=c, repetitions=reps, trim_fraction=trim_fraction,
                         seed=seed, timing_recorded=with_timing, exact_p_star=exact.p_star,
                         exact_lag_seconds=list(exact.per_lag_seconds), exact_taus=list(exact.pacf.taus),
                         lsar=_summarize("lsar", exact, lsar_runs, trim_fraction),
                         rh=_summarize("rh", exact, rh_runs, trim_fraction))


def run_sweep(series: TimeSeries, c_list, p_bar: int, reps: int, trim_fraction: float, seed: int,
              with_timing: bool = True, *, workers: int = 8) -> list:
    """bench.cpp:214-243: per c, `reps` LSAR and RH fits against one exact
    fit (seeds derive_seed(seed, (ci << 20) + 0x10000 / 0x20000 + r)); rows
    carry the max-over-lags mean lag time and trimmed error."""
    c_list = list(c_list)
    if not c_list:
        raise UsageError("empty c list")
    exact = exact_fit(series, p_bar)
    rows = []
    for ci, c in enumerate(c_list):
        for method in ("lsar", "rh"):
            tag = 0x10000 if method == "lsar" else 0x20000
            seeds = [derive_seed(seed, (ci << 20) + tag + r) for r in range(reps)]
            runs = (_lsar_reps(series, p_bar, c, seeds, workers) if method == "lsar"
                    else fit_many([series] * reps, method, p_bar, c, seeds, workers=workers))
            if not with_timing:
                for f in runs:
                    _strip_timing(f)
            sm = _summarize(method, exact, runs, trim_fraction)
            rows.append(SweepRow(method, int(c), max(sm.mean_lag_seconds), max(sm.trimmed_error_pct)))
    return rows


def compare_to_json(r: CompareReport) -> str:
    """bench.cpp:286-303 (nlohmann objects: keys sorted, dump(2))."""
    def mc(m: MethodComparison):
        return {"method": m.method, "trimmed_error_pct": m.trimmed_error_pct, "mean_lag_seconds": m.mean_lag_seconds,
                "mean_upfront_seconds": m.mean_upfront_seconds, "p_stars": m.p_stars}
    j = {"n": r.n, "p_bar": r.p_bar, "c": r.c, "repetitions": r.repetitions, "trim_fraction": r.trim_fraction,
         "seed": r.seed, "timing_recorded": r.timing_recorded,
         "exact": {"p_star": r.exact_p_star, "per_lag_seconds": r.exact_lag_seconds, "taus": r.exact_taus},
         "lsar": mc(r.lsar), "rh": mc(r.rh)}
    return json.dumps(j, indent=2, sort_keys=True) + "\n"



# ---------------------------------------------------------------------------
# Report writers (bench.cpp:301-363, toeplitz.cpp:148-158): same text, %.17g
def _write_text(path: str, text: str) -> None:
    try:
        with open(path, "w", newline="") as f:
            f.write(text)
    except OSError:
        raise DataError("cannot write " + path) from None


def write_run_report(report: RunReport, path: str) -> None:
    _write_text(path, report_to_json(report))


def write_compare_json(report: CompareReport, path: str) -> None:
    _write_text(path, compare_to_json(report))


def write_compare_errors_csv(report: CompareReport, path: str) -> None:
    lines = ["lag,lsar_error,rh_error\n"]
    for h, (a, b) in enumerate(zip(report.lsar.trimmed_error_pct, report.rh.trimmed_error_pct)):
        lines.append("%d,%.17g,%.17g\n" % (h + 1, a, b))
    _write_text(path, "".join(lines))


def write_compare_timing_csv(report: CompareReport, path: str) -> None:
    lines = ["lag,exact_cum,lsar_cum,rh_cum\n"]
    ex = ls = 0.0
    rh = report.rh.mean_upfront_seconds
    for h in range(len(report.exact_lag_seconds)):
        ex += report.exact_lag_seconds[h]
        ls += report.lsar.mean_lag_seconds[h]
        rh += report.rh.mean_lag_seconds[h]
        lines.append("%d,%.17g,%.17g,%.17g\n" % (h + 1, ex, ls, rh))
    _write_text(path, "".join(lines))


def write_sweep_csv(rows, path: str) -> None:
    lines = ["method,c,max_seconds,max_error_pct\n"]
    for r in rows:
        lines.append("%s,%d,%.17g,%.17g\n" % (r.method, r.c, r.max_lag_seconds, r.max_error_pct))
    _write_text(path, "".join(lines))


def write_pacf_plot_csv(pacf: PACFResult, path: str) -> None:
    lines = ["lag,tau,bound_hi,bound_lo\n"]
    for i, t in enumerate(pacf.taus):
        lines.append("%d,%.17g,%.17g,%.17g\n" % (i + 1, t, pacf.bound, -pacf.bound))
    _write_text(path, "".join(lines))


def write_pacf_csv(pacf: PACFResult, path: str) -> None:
    lines = ["lag,tau,bound\n"]
    for i, t in enumerate(pacf.taus):
        lines.append("%d,%.17g,%.17g\n" % (i + 1, t, pacf.bound))
    _write_text(path, "".join(lines))
