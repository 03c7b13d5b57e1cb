/*
 * toepfit_b200.h -- C ABI of the B200-native LSAR / Repeated-Halving order
 * sweep (arXiv 2112.12994).  Drop-in for the reference's hot-path entry
 * points (namespace toepfit, /root/reference/proj):
 *
 *   tf_upload_series   <- TimeSeries(std::vector<double>)      series.hpp:16-31, series.cpp:23-32
 *   tf_lsar_sweep      <- FitResult lsar_fit(series, p_bar, c, seed)          lsar.hpp:89, lsar.cpp:100-124
 *   tf_lsar_sweep_batch<- lsar_fit over many series / seeds (the run_compare / bench.cpp:183-188, 221-228
 *                         run_sweep loops; BASELINE C5 batch)
 *   tf_rh_sweep        <- FitResult rh_fit(series, p_bar, c, cfg*, seed)      repeated_halving.hpp:97-99,
 *                                                                            repeated_halving.cpp:191-232
 *   tf_residuals       <- Eigen::VectorXd residuals(sys, phi)                 toeplitz.hpp:84-86, toeplitz.cpp:87-98
 *   tf_sample_rows     <- SampleSet sample_rows(pi, c, seed)                  sketch.hpp:47-48, sketch.cpp:20-59
 *   tf_apply_sample    <- apply_sample(sys, sample, width, A_S, b_S)          sketch.hpp:53-54, sketch.cpp:61-79
 *   tf_solve_sampled   <- solve_compressed(apply_sample(...))                 sketch.hpp:63-64, sketch.cpp:96-101
 *   tf_select_order    <- int select_order(const PACFResult&)                 toeplitz.hpp:100, toeplitz.cpp:133-138
 *   tf_exact_sweep     <- exact per-lag OLS fit (run_fit "exact")              bench.cpp:27-48
 *   tf_srht_sweep      <- FitResult srht_fit(series, p_bar, c, seed)          bench.cpp:50-72, sketch.cpp:187-239
 *   tf_hadamard        <- void hadamard_apply(std::span<double>)              sketch.hpp, sketch.cpp:107-120
 *
 * Conventions (mirroring the reference): indices are 0-based int64, series
 * and coefficients are fp64; errors never cross the ABI as exceptions --
 * every call returns a tf_status (USAGE/DATA/NUMERICAL mirror UsageError /
 * DataError / NumericalError of errors.hpp:12-29, CLI exit codes 2/3/4) and
 * tf_last_error() holds the message.  The caller owns every host buffer; the
 * context owns device memory.  One context per host thread (the reference is
 * single-threaded; distinct fits may run concurrently on distinct contexts,
 * SPEC.md:431).  Nothing here falls back to the CPU: without a usable CUDA
 * device tf_create returns TF_CUDA.
 */
#ifndef TOEPFIT_B200_H
#define TOEPFIT_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  TF_OK = 0,
  TF_USAGE = 1,
  TF_DATA = 2,
  TF_NUMERICAL = 3,
  TF_CUDA = 4,
  TF_NCCL = 5
} tf_status;

typedef struct tf_context tf_context;

typedef struct {
  int device;    /* CUDA device ordinal */
  int priority;  /* stream priority: 0 = default, k > 0 = k levels above it (clamped to the
                    device range) -- lets a latency-bound fit run ahead of concurrent ones.
                    The default is one step above the device's lowest priority, which the
                    context's second stream takes (the FFT lags' score updates, which run
                    beside the lag's solve and must yield the SMs to it) */
} tf_opts;

/* RHConfig (repeated_halving.hpp:56-65) */
typedef struct {
  int64_t base_threshold;
  int64_t sample_count;
  int64_t gaussian_rows;
  uint64_t seed;
} tf_rh_cfg;

/* Optional diagnostics / deterministic-index mode for the LSAR sweep.  All
 * pointers are host pointers and may be NULL. */
typedef struct {
  const int64_t* fixed_idx; /* [p_bar][c]: replaces sampling (deterministic-index mode) */
  const double* fixed_w;    /* [p_bar][c]; NULL with fixed_idx: each lag's own weights
                               1/sqrt(c pi_i) from its distribution (sketch.cpp:56-57) */
  int64_t* idx_out;         /* [p_bar][c] drawn indices */
  double* w_out;            /* [p_bar][c] drawn weights */
  double* rnorm2_out;       /* [p_bar] ||r_p||^2 */
  double* ssum_out;         /* [p_bar] sum of the scores sampled at lag p */
  double* scores_out;       /* [n - p_bar] scores of the last lag */
  double* resid_out;        /* [n - p_bar] residuals of the last lag */
  int* method_out;          /* [p_bar] SolveMethod of the lag (toeplitz.hpp:49-56): 0 exact_qr (CPQR
                               rank = p), 1 exact_svd (rank < p: minimum-norm SVD answer) */
  double* phase_seconds;    /* [p_bar][3] device time of sampling, solve, fused pass */
  int64_t* launches_out;    /* kernel launches issued by the sweep */
  int* rank_out;            /* [p_bar] CPQR rank of the sampled system (threshold max(c, p) eps) */
  int* svd_sweeps_out;      /* [p_bar] Jacobi sweeps of the minimum-norm SVD (0 for exact_qr lags) */
} tf_lsar_diag;

typedef struct {
  const int64_t* fixed_idx;     /* [p_bar][c] per-lag samples (nullable) */
  const double* fixed_w;        /* [p_bar][c]; NULL with fixed_idx: weights from the final scores */
  const int64_t* fixed_levels;  /* concatenated halving index sets, levels 1..depth (nullable) */
  const int64_t* fixed_up_idx;  /* [depth][sample_count] upward-pass samples (nullable) */
  const double* fixed_up_w;
  double* scores_out;           /* [n - p_bar] final leverage scores */
  int* depth_out;
  int64_t* idx_out;             /* [p_bar][c] */
  double* w_out;
  int64_t* levels_out;          /* concatenated halving index sets, levels 1..depth */
  int64_t* up_idx_out;          /* [depth][sample_count] upward-pass positions */
  double* up_w_out;             /* [depth][sample_count] upward-pass weights */
  int64_t* launches_out;        /* kernel launches issued by the sweep */
  int* method_out;              /* [p_bar] 0 exact_qr / 1 exact_svd (as tf_lsar_diag) */
  int* rank_out;                /* [p_bar] CPQR rank */
} tf_rh_diag;

const char* tf_version(void);
tf_status tf_create(const tf_opts* opts, tf_context** out);
void tf_destroy(tf_context* ctx);
const char* tf_last_error(const tf_context* ctx);

/* Series resident in HBM for the following sweeps.  Validates non-empty and
 * finite values (DataError, series.cpp:23-32). */
tf_status tf_upload_series(tf_context* ctx, const double* y, int64_t n);
/* Synthetic AR series generated on the device into the context (the BASELINE
 * root-based cascade generator: x_t = x_{t-1} / r_k + in_t per real root r_k,
 * counter-RNG innovations, innovations 0 = N(0,1), 1 = Student-t(3)/sqrt(3);
 * the first burn_in samples are dropped).  Replaces host generation +
 * upload for large configs. */
tf_status tf_generate_series(tf_context* ctx, const double* roots, int q, int64_t n, uint64_t seed,
                             int innovations, int64_t burn_in);
/* Copy the first n values of the resident series to the host. */
tf_status tf_download_series(tf_context* ctx, double* out, int64_t n);
/* Same, from a device pointer already in HBM (no host copy). */
tf_status tf_upload_series_device(tf_context* ctx, const double* d_y, int64_t n);

/* LSAR order sweep p = 1..p_bar on the uploaded series.  Outputs (host):
 * taus[p_bar], coefs_packed[p_bar (p_bar+1)/2] (phi_1, phi_2, ...),
 * lag_seconds[p_bar] (device time per lag body), p_star (nullable ok). */
tf_status tf_lsar_sweep(tf_context* ctx, int p_bar, int64_t c, uint64_t seed,
                        const tf_lsar_diag* diag, double* taus, double* coefs_packed,
                        double* lag_seconds, int* p_star);

/* One lag of the LSAR recursion: LsarDriver::first_lag (p = 1) and
 * LsarDriver::advance (p > 1) (lsar.hpp:65-84, lsar.cpp:70-98).  For p > 1 the
 * lag-(p-1) state is scores_in / resid_in (w = n - p_bar host values each), or
 * both NULL to continue from the state the previous tf_lsar_step call left on
 * the device.  Outputs (nullable): the lag-p scores (the distribution's
 * weights at lag p), residuals (w each), phi (p values, reference order) and
 * the solve method.  Errors as lsar_fit; TF_USAGE for p outside 1..p_bar
 * ("cannot advance past maximum lag"). */
tf_status tf_lsar_step(tf_context* ctx, int p_bar, int64_t c, uint64_t seed, int p, const double* scores_in,
                       const double* resid_in, double* scores_out, double* resid_out, double* phi_out,
                       int* method_out);

/* LSAR order sweeps of a BATCH of independent fits in one pass per lag:
 * series b = y + b * y_stride (n values each; y_stride 0: one series shared
 * by every fit, i.e. B seeds over one series), seed seeds[b], all with the
 * same p_bar (<= 63) and c.  fixed_idx / fixed_w (nullable, [batch][p_bar][c])
 * replace the draws (deterministic-index mode).  Outputs per fit b:
 * taus[b * p_bar ..], coefs_packed[b * p_bar (p_bar+1)/2 ..], p_star[b],
 * status_out[3 b ..] = {error code (0, 1 usage, 2 data, 3 numerical), lag,
 * reason}; lag_seconds[p_bar] is the batch's device time per lag.  Each fit
 * equals lsar_fit(series_b, p_bar, c, seeds[b]) (lsar.cpp:100-124); a fit
 * whose sampled system breaks down is re-run through tf_lsar_sweep. */
tf_status tf_lsar_sweep_batch(tf_context* ctx, const double* y, int64_t y_stride, int64_t batch, int64_t n,
                              int p_bar, int64_t c, const uint64_t* seeds, const int64_t* fixed_idx,
                              const double* fixed_w, double* taus, double* coefs_packed, double* lag_seconds,
                              int* p_star, int* status_out);

/* Repeated-Halving sweep; cfg NULL -> RHConfig::defaults(n - p_bar, p_bar + 1, c,
 * derive_seed(seed, 0x5c07e5)). */
tf_status tf_rh_sweep(tf_context* ctx, int p_bar, int64_t c, const tf_rh_cfg* cfg, uint64_t seed,
                      const tf_rh_diag* diag, double* taus, double* coefs_packed,
                      double* lag_seconds, double* upfront_seconds, int* p_star);

/* ---- Repeated Halving over a general row source ----
 * RowSource (repeated_halving.hpp:17-23): an n x k matrix reached through
 * gather(user, idx, count, out), which writes rows idx[0..count) into out
 * (count x k, row-major, host memory). */
typedef void (*tf_gather_fn)(void* user, const int64_t* idx, int64_t count, double* out);
/* generalized_leverage (repeated_halving.hpp:76-78, repeated_halving.cpp:54-123):
 * leverage of the rows of C (rows x c_cols, row-major) through the column space
 * of B (brows x b_cols): ||R^-T P^T x||^2 (sketch_rows 0) or its sketch with
 * sketch_rows Gaussian mixes from Rng(sketch_seed).  Errors: TF_USAGE column
 * count mismatch; TF_NUMERICAL brows < k ("too few rows") or B rank deficient
 * under the CPQR rule (threshold max(brows, k) eps). */
tf_status tf_generalized_leverage(tf_context* ctx, const double* c_rows, int64_t rows, int64_t c_cols, const double* b,
                                  int64_t brows, int64_t b_cols, int64_t sketch_rows, uint64_t sketch_seed, double* out);
/* repeated_halving(RowSource, RHConfig) (repeated_halving.cpp:126-180): the
 * downward halving (bit-identical level sets), the sketched upward pass; the
 * approximation's rows (approx_rows x k, row-major) land in approx_out
 * (capacity approx_cap rows), levels = halving depth. */
tf_status tf_repeated_halving(tf_context* ctx, int64_t n, int64_t k, tf_gather_fn gather, void* user,
                              const tf_rh_cfg* cfg, double* approx_out, int64_t approx_cap, int64_t* approx_rows,
                              int* levels);

/* Exact per-lag OLS on the full series (bench.cpp:27-48, the reference's
 * "exact" method): lag h uses all n - h rows.  Outputs as tf_lsar_sweep;
 * p_star uses the bound 1.96 / sqrt(n - p_bar). */
tf_status tf_exact_sweep(tf_context* ctx, int p_bar, double* taus, double* coefs_packed, double* lag_seconds,
                         int* p_star);

/* Subsampled randomized Hadamard transform sweep (bench.cpp:50-72 srht_fit;
 * sketch.cpp:187-239 srht_solve per lag with seed derive_seed(seed, h)).
 * Outputs as tf_lsar_sweep; p_star uses the bound 1.96 / sqrt(c).  Errors:
 * TF_USAGE for p_bar < 1 or c < p_bar, TF_DATA for n <= p_bar + 1. */
tf_status tf_srht_sweep(tf_context* ctx, int p_bar, int64_t c, uint64_t seed, double* taus, double* coefs_packed,
                        double* lag_seconds, int* p_star);

/* In-place orthonormal Walsh-Hadamard transform of a host vector of
 * power-of-two length (sketch.cpp:107-120; TF_USAGE otherwise). */
tf_status tf_hadamard(tf_context* ctx, double* x, int64_t n);

/* ---- single operations on host buffers (tests, integration) ---- */
tf_status tf_residuals(tf_context* ctx, const double* y, int64_t n_used, int p, const double* phi,
                       double* r_out);
/* Draw c rows from the distribution pi (sketch.cpp:20-59): TF_DATA for a
 * negative entry or |sum pi - 1| > 1e-8 (sketch.cpp:25-32), TF_USAGE for c < 1. */
tf_status tf_sample_rows(tf_context* ctx, const double* pi, int64_t n, int64_t c, uint64_t seed,
                         int64_t* idx_out, double* w_out);
/* A_S (c x width, row-major) and b_S of the window system (y, n_used, p). */
tf_status tf_apply_sample(tf_context* ctx, const double* y, int64_t n_used, int p,
                          const int64_t* idx, const double* w, int64_t c, int width, double* a_out,
                          double* b_out);
/* phi = argmin || A_S phi - b_S || for the sampled window system
 * (solve_compressed, sketch.cpp:96-101 -> toeplitz.cpp:57-85): method_out 0 =
 * exact_qr (CPQR rank = p), 1 = exact_svd (minimum-norm answer). */
tf_status tf_solve_sampled(tf_context* ctx, const double* y, int64_t n_used, int p,
                           const int64_t* idx, const double* w, int64_t c, double* phi_out,
                           int* method_out);

int tf_select_order(const double* taus, int p_bar, double bound);
/* Diagnostics: measured fp64 FMA throughput of this device (TFLOP/s) from a
 * DFMA microbenchmark, the denominator of the fp64 roofline. */
tf_status tf_probe_fp64_peak(tf_context* ctx, double* tflops);

/* Diagnostics: the first lag q of a p_bar sweep whose pass runs the FFT FIR
 * (k_lsar_pass_fft); lags below it run the direct tensor-core FIR.  p_bar + 1
 * when the sweep takes no FFT lag.  (No reference counterpart: an execution
 * detail the bench needs for the per-kernel roofline.) */
tf_status tf_fft_first_lag(tf_context* ctx, int p_bar, int* lag);

/* ---- row-sharded LSAR sweep of one long series (one process per GPU;
 *      SURVEY.md 8(e); BASELINE C3 2-GPU, C4 1/2/4/8 GPUs) ----
 * Rank g holds the window rows [row0_g, row0_g + w_g) of the global window
 * (w = n - p_bar, contiguous balanced blocks) as the slice
 * y[row0_g .. row0_g + w_g + p_bar) -- uploaded with tf_upload_series, or
 * generated whole with tf_generate_series and cut with tf_keep_slice.  The
 * communicator: rank 0 calls tf_nccl_unique_id, the caller broadcasts the
 * bytes, every rank calls tf_nccl_init.  tf_lsar_sweep_sharded then runs the
 * lag loop with NCCL on the context stream (no host round trips; graph
 * captured): per lag an allgather of every shard's (sum s, sum r^2) -- the
 * global ||r||^2 and the shards' CDF segments (prefix in rank order); each
 * rank resolves the draws of Rng(derive_seed(seed, p)) in its segment; an
 * allgather of the shards' double-double Gram partials, summed in rank order,
 * so every rank runs the same rank-revealing solve and holds the same phi.
 * The result equals lsar_fit on the whole series up to the summation order of
 * the reductions (lsar.cpp:100-124).  Outputs as tf_lsar_sweep (on every rank);
 * diag: rnorm2 / ssum / method / rank / phases / launches (fixed-index mode is
 * single-shard only). */
tf_status tf_nccl_unique_id(unsigned char* out, int bytes);  /* bytes >= 128 (ncclUniqueId) */
tf_status tf_nccl_init(tf_context* ctx, const unsigned char* id, int world, int rank);
tf_status tf_keep_slice(tf_context* ctx, int64_t start, int64_t len);
tf_status tf_lsar_sweep_sharded(tf_context* ctx, int p_bar, int64_t c, uint64_t seed, const tf_lsar_diag* diag,
                                double* taus, double* coefs_packed, double* lag_seconds, int* p_star);
int64_t tf_tpu_size(int K);

/* Device-time span of ctx's last sweep relative to the start of ref's last
 * sweep (ms, CUDA events): for timing concurrent sweeps on several contexts
 * (independent fits may run concurrently). */
tf_status tf_sweep_span(const tf_context* ref, const tf_context* ctx, double* start_ms, double* end_ms);
uint64_t tf_derive_seed(uint64_t seed, uint64_t tag);

#ifdef __cplusplus
}
#endif

#endif
