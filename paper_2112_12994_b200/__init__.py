"""paper_2112_12994_b200 -- B200-native LSAR / Repeated-Halving order sweep.

Host mirror of the reference toepfit API over the C ABI of
libtoepfit_b200.so (hand-written sm_100a kernels); see DESIGN.md.
"""
from .api import (CudaError, DataError, Engine, FitResult, NumericalError, PACFResult, RHConfig,  # noqa: F401
                  LeverageState, LsarDriver, GaussianSketch, RowSource, DenseRowSource, AugmentedRowSource,
                  SpectralApprox, generalized_leverage, repeated_halving, rh_leverage_scores,
                  RunReport, TimeSeries, UsageError, default_engine, derive_seed, lsar_fit, lsar_fit_batch,
                  report_to_json, rh_fit, run_fit, select_order, exact_fit, fit_many,
                  load_series_bin, save_series_bin, srht_fit, hadamard_apply,
                  srht_sample_count, SrhtCount, run_compare, run_sweep, compare_to_json,
                  CompareReport, MethodComparison, SweepRow, relative_error_pct, trimmed_mean,
                  write_run_report, write_compare_json, write_compare_errors_csv, write_compare_timing_csv,
                  write_sweep_csv, write_pacf_plot_csv, write_pacf_csv)

__all__ = ["TimeSeries", "FitResult", "PACFResult", "RHConfig", "RunReport", "Engine", "LeverageState", "LsarDriver", "GaussianSketch", "RowSource",
           "DenseRowSource", "AugmentedRowSource", "SpectralApprox", "generalized_leverage", "repeated_halving",
           "rh_leverage_scores",
           "UsageError", "DataError", "NumericalError", "CudaError", "lsar_fit", "lsar_fit_batch", "rh_fit",
           "run_fit", "report_to_json", "select_order", "derive_seed", "default_engine",
           "exact_fit", "fit_many", "load_series_bin", "save_series_bin", "srht_fit",
           "hadamard_apply", "srht_sample_count", "SrhtCount", "run_compare", "run_sweep",
           "compare_to_json", "CompareReport", "MethodComparison", "SweepRow", "relative_error_pct",
           "trimmed_mean", "write_run_report", "write_compare_json", "write_compare_errors_csv",
           "write_compare_timing_csv", "write_sweep_csv", "write_pacf_plot_csv", "write_pacf_csv"]
