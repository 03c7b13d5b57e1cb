"""ctypes binding of the C ABI in include/toepfit_b200.h.

The product path is the in-tree libtoepfit_b200.so (hand-written sm_100a
kernels).  There is no fallback: if the library is missing or no CUDA device
is usable, every entry point raises.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libtoepfit_b200.so")

TF_OK, TF_USAGE, TF_DATA, TF_NUMERICAL, TF_CUDA, TF_NCCL = range(6)

_f64p = C.POINTER(C.c_double)
_i64p = C.POINTER(C.c_int64)
_i32p = C.POINTER(C.c_int)


class TfOpts(C.Structure):
    _fields_ = [("device", C.c_int), ("priority", C.c_int)]


class TfRhCfg(C.Structure):
    _fields_ = [("base_threshold", C.c_int64), ("sample_count", C.c_int64),
                ("gaussian_rows", C.c_int64), ("seed", C.c_uint64)]


class TfLsarDiag(C.Structure):
    _fields_ = [("fixed_idx", _i64p), ("fixed_w", _f64p), ("idx_out", _i64p), ("w_out", _f64p),
                ("rnorm2_out", _f64p), ("ssum_out", _f64p), ("scores_out", _f64p),
                ("resid_out", _f64p), ("method_out", _i32p), ("phase_seconds", _f64p),
                ("launches_out", _i64p), ("rank_out", _i32p), ("svd_sweeps_out", _i32p)]


class TfRhDiag(C.Structure):
    _fields_ = [("fixed_idx", _i64p), ("fixed_w", _f64p), ("fixed_levels", _i64p),
                ("fixed_up_idx", _i64p), ("fixed_up_w", _f64p), ("scores_out", _f64p),
                ("depth_out", _i32p), ("idx_out", _i64p), ("w_out", _f64p),
                ("levels_out", _i64p), ("up_idx_out", _i64p), ("up_w_out", _f64p),
                ("launches_out", _i64p), ("method_out", _i32p), ("rank_out", _i32p)]


# RowSource gather callback (tf_gather_fn): (user, idx, count, out rows x k row-major)
GATHER_FN = C.CFUNCTYPE(None, C.c_void_p, C.POINTER(C.c_int64), C.c_int64, C.POINTER(C.c_double))

EXPORTS = [
    "tf_version", "tf_create", "tf_destroy", "tf_last_error", "tf_upload_series",
    "tf_upload_series_device", "tf_lsar_sweep", "tf_rh_sweep", "tf_residuals", "tf_sample_rows",
    "tf_apply_sample", "tf_solve_sampled", "tf_select_order", "tf_derive_seed",
    "tf_probe_fp64_peak", "tf_fft_first_lag", "tf_nccl_unique_id", "tf_nccl_init", "tf_keep_slice", "tf_lsar_sweep_sharded",
    "tf_tpu_size", "tf_sweep_span", "tf_exact_sweep", "tf_srht_sweep", "tf_hadamard", "tf_generate_series", "tf_download_series",
    "tf_lsar_sweep_batch", "tf_lsar_step", "tf_generalized_leverage", "tf_repeated_halving",
]

_lib = None


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
            " (there is no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    L.tf_version.restype = C.c_char_p
    L.tf_last_error.restype = C.c_char_p
    L.tf_last_error.argtypes = [C.c_void_p]
    L.tf_create.argtypes = [C.POINTER(TfOpts), C.POINTER(C.c_void_p)]
    L.tf_destroy.argtypes = [C.c_void_p]
    L.tf_upload_series.argtypes = [C.c_void_p, _f64p, C.c_int64]
    L.tf_upload_series_device.argtypes = [C.c_void_p, C.c_void_p, C.c_int64]
    L.tf_lsar_sweep.argtypes = [C.c_void_p, C.c_int, C.c_int64, C.c_uint64, C.POINTER(TfLsarDiag),
                                _f64p, _f64p, _f64p, _i32p]
    L.tf_rh_sweep.argtypes = [C.c_void_p, C.c_int, C.c_int64, C.POINTER(TfRhCfg), C.c_uint64,
                              C.POINTER(TfRhDiag), _f64p, _f64p, _f64p, _f64p, _i32p]
    L.tf_residuals.argtypes = [C.c_void_p, _f64p, C.c_int64, C.c_int, _f64p, _f64p]
    L.tf_sample_rows.argtypes = [C.c_void_p, _f64p, C.c_int64, C.c_int64, C.c_uint64, _i64p, _f64p]
    L.tf_apply_sample.argtypes = [C.c_void_p, _f64p, C.c_int64, C.c_int, _i64p, _f64p, C.c_int64,
                                  C.c_int, _f64p, _f64p]
    L.tf_solve_sampled.argtypes = [C.c_void_p, _f64p, C.c_int64, C.c_int, _i64p, _f64p, C.c_int64,
                                   _f64p, _i32p]
    L.tf_select_order.argtypes = [_f64p, C.c_int, C.c_double]
    L.tf_select_order.restype = C.c_int
    L.tf_derive_seed.argtypes = [C.c_uint64, C.c_uint64]
    L.tf_derive_seed.restype = C.c_uint64
    L.tf_probe_fp64_peak.argtypes = [C.c_void_p, _f64p]
    L.tf_fft_first_lag.argtypes = [C.c_void_p, C.c_int, _i32p]
    L.tf_nccl_unique_id.argtypes = [C.c_char_p, C.c_int]
    L.tf_nccl_init.argtypes = [C.c_void_p, C.c_char_p, C.c_int, C.c_int]
    L.tf_keep_slice.argtypes = [C.c_void_p, C.c_int64, C.c_int64]
    L.tf_lsar_sweep_sharded.argtypes = [C.c_void_p, C.c_int, C.c_int64, C.c_uint64, C.POINTER(TfLsarDiag),
                                        _f64p, _f64p, _f64p, _i32p]
    _u64p = C.POINTER(C.c_uint64)
    L.tf_generate_series.argtypes = [C.c_void_p, _f64p, C.c_int, C.c_int64, C.c_uint64, C.c_int, C.c_int64]
    L.tf_download_series.argtypes = [C.c_void_p, _f64p, C.c_int64]
    L.tf_lsar_sweep_batch.argtypes = [C.c_void_p, _f64p, C.c_int64, C.c_int64, C.c_int64, C.c_int, C.c_int64, _u64p,
                                      _i64p, _f64p, _f64p, _f64p, _f64p, _i32p, _i32p]
    L.tf_exact_sweep.argtypes = [C.c_void_p, C.c_int, _f64p, _f64p, _f64p, _i32p]
    L.tf_srht_sweep.argtypes = [C.c_void_p, C.c_int, C.c_int64, C.c_uint64, _f64p, _f64p, _f64p, _i32p]
    L.tf_hadamard.argtypes = [C.c_void_p, _f64p, C.c_int64]
    L.tf_sweep_span.argtypes = [C.c_void_p, C.c_void_p, _f64p, _f64p]
    L.tf_version.argtypes = []
    L.tf_generalized_leverage.argtypes = [C.c_void_p, _f64p, C.c_int64, C.c_int64, _f64p, C.c_int64, C.c_int64,
                                          C.c_int64, C.c_uint64, _f64p]
    L.tf_repeated_halving.argtypes = [C.c_void_p, C.c_int64, C.c_int64, GATHER_FN, C.c_void_p, C.POINTER(TfRhCfg),
                                      _f64p, C.c_int64, _i64p, _i32p]
    L.tf_lsar_step.argtypes = [C.c_void_p, C.c_int, C.c_int64, C.c_uint64, C.c_int, _f64p, _f64p, _f64p, _f64p,
                               _f64p, _i32p]
    L.tf_tpu_size.argtypes = [C.c_int]
    L.tf_tpu_size.restype = C.c_int64
    for name in EXPORTS:
        if not hasattr(L, name):
            raise RuntimeError(f"{LIB_PATH} does not export {name}")
        if name not in ("tf_version",) and getattr(L, name).argtypes is None:
            raise RuntimeError(f"{name}: no ctypes signature (64-bit arguments would be truncated)")
    _lib = L
    return L


def ptr(a, t=_f64p):
    return None if a is None else a.ctypes.data_as(t)
