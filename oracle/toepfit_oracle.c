/*
 * toepfit_oracle.c -- Eigen-free CPU restatement of the reference hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see toepfit_oracle.h).  Each function cites the
 * reference file:line it restates (paths relative to /root/reference/proj).
 * Compiled with -ffp-contract=off: every fused multiply-add below is an
 * explicit fma() call, so the operation order is fixed and documented.
 */
#define _POSIX_C_SOURCE 200809L
#include "toepfit_oracle.h"

#include <float.h>
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

static _Thread_local char g_err[512];

const char* orc_last_error(void) { return g_err; }

static int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
  return code;
}

static double now_seconds(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

#define XMALLOC(T, n) ((T*)malloc(sizeof(T) * (size_t)((n) > 0 ? (n) : 1)))

/* ======================================================================
 * RNG -- rng.hpp:14-84 (Weyl increment + splitmix64 finalizer)
 * ==================================================================== */
#define GOLDEN 0x9e3779b97f4a7c15ull

uint64_t orc_mix(uint64_t z) { /* rng.hpp:69-73 */
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

void orc_rng_init(orc_rng* r, uint64_t seed) {
  r->state = seed;
  r->spare = 0.0;
  r->has_spare = 0;
}

uint64_t orc_rng_next(orc_rng* r) { /* rng.hpp:23-26 */
  r->state += GOLDEN;
  return orc_mix(r->state);
}

orc_rng orc_rng_fork(const orc_rng* r, uint64_t tag) { /* rng.hpp:30-32 */
  orc_rng out;
  orc_rng_init(&out, orc_mix(r->state ^ orc_mix(tag + 0x632be59bd9b4e019ull)));
  return out;
}

double orc_rng_uniform01(orc_rng* r) { /* rng.hpp:35 */
  return (double)(orc_rng_next(r) >> 11) * 0x1.0p-53;
}

static double rng_uniform(orc_rng* r, double lo, double hi) { /* rng.hpp:37 */
  return lo + (hi - lo) * orc_rng_uniform01(r);
}

double orc_rng_normal(orc_rng* r) { /* rng.hpp:41-56, polar method with cached spare */
  if (r->has_spare) {
    r->has_spare = 0;
    return r->spare;
  }
  double u, v, s;
  do {
    u = rng_uniform(r, -1.0, 1.0);
    v = rng_uniform(r, -1.0, 1.0);
    s = u * u + v * v; /* no contraction: (u*u) rounded, (v*v) rounded, then added */
  } while (s >= 1.0 || s == 0.0);
  const double f = sqrt(-2.0 * log(s) / s);
  r->spare = v * f;
  r->has_spare = 1;
  return u * f;
}

uint64_t orc_rng_below(orc_rng* r, uint64_t bound) { /* rng.hpp:59-66 */
  const uint64_t mx = ~(uint64_t)0;
  const uint64_t limit = mx - mx % bound;
  uint64_t x;
  do {
    x = orc_rng_next(r);
  } while (x >= limit);
  return x % bound;
}

/* OpenMP thread count of the parallel loops (row / column independent: the
 * results do not depend on it).  bench.py's single-core CPU baseline sets 1. */
#include <omp.h>
void orc_set_threads(int n) { omp_set_num_threads(n > 0 ? n : 1); }
int orc_max_threads(void) { return omp_get_max_threads(); }

uint64_t orc_derive_seed(uint64_t seed, uint64_t tag) { /* rng.hpp:82-84 */
  orc_rng r;
  orc_rng_init(&r, seed);
  orc_rng f = orc_rng_fork(&r, tag);
  return orc_rng_next(&f);
}

/* ======================================================================
 * small dense helpers (fixed summation order)
 * ==================================================================== */
static double dot(const double* a, const double* b, int64_t n) {
  double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
  int64_t i = 0;
  for (; i + 4 <= n; i += 4) {
    s0 = fma(a[i], b[i], s0);
    s1 = fma(a[i + 1], b[i + 1], s1);
    s2 = fma(a[i + 2], b[i + 2], s2);
    s3 = fma(a[i + 3], b[i + 3], s3);
  }
  for (; i < n; ++i) s0 = fma(a[i], b[i], s0);
  return (s0 + s1) + (s2 + s3);
}

static double sqnorm(const double* a, int64_t n) { return dot(a, a, n); }

static void axpy(double alpha, const double* x, double* y, int64_t n) {
  for (int64_t i = 0; i < n; ++i) y[i] = fma(alpha, x[i], y[i]);
}

static int cmp_i64(const void* a, const void* b) {
  const int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
  return (x > y) - (x < y);
}

/* ======================================================================
 * toeplitz.cpp:87-98 -- streaming residuals r = X_p phi - y[p..]
 * Per-tap axpy in tap order j = 0..p-1 starting from -y (fma each step).
 * ==================================================================== */
int orc_residuals(const double* y, int64_t n_used, int p, const double* phi, double* r) {
  if (p < 1) return fail(ORC_USAGE, "lag order must be at least 1");
  if (n_used <= p) return fail(ORC_DATA, "series window too short for lag order");
  const int64_t m = n_used - p;
  /* row blocks are independent: every r[i] sees the same fma sequence as the
   * reference's whole-vector tap loop, whatever the thread count */
  const int64_t blk = 4096;
#pragma omp parallel for schedule(static)
  for (int64_t b0 = 0; b0 < m; b0 += blk) {
    const int64_t b1 = b0 + blk < m ? b0 + blk : m;
    for (int64_t i = b0; i < b1; ++i) r[i] = -y[p + i];
    for (int j = 0; j < p; ++j) {
      const double a = phi[j];
      const double* src = y + (p - 1 - j);
      for (int64_t i = b0; i < b1; ++i) r[i] = fma(a, src[i], r[i]);
    }
  }
  return ORC_OK;
}

/* ======================================================================
 * lsar.cpp:11-36
 * ==================================================================== */
static double seq_sqnorm(const double* x, int64_t n) {
  double s = 0.0;
  for (int64_t i = 0; i < n; ++i) s += x[i] * x[i];
  return s;
}

int orc_init_leverage_p1(const double* window, int64_t w, double* out) {
  const double total = seq_sqnorm(window, w);
  if (total == 0.0) return fail(ORC_NUMERICAL, "all-zero window; leverage undefined");
  for (int64_t i = 0; i < w; ++i) out[i] = (window[i] * window[i]) / total;
  return ORC_OK;
}

int orc_leverage_update(const double* scores, const double* r, int64_t w, double* out) {
  const double total = seq_sqnorm(r, w);
  if (total == 0.0)
    return fail(ORC_NUMERICAL, "zero residual norm; sampling distribution undefined");
  for (int64_t i = 0; i < w; ++i) out[i] = scores[i] + (r[i] * r[i]) / total;
  return ORC_OK;
}

int orc_leverage_to_distribution(const double* scores, int64_t w, double* out) {
  if (w == 0) return fail(ORC_USAGE, "empty score vector");
  double total = 0.0;
  for (int64_t i = 0; i < w; ++i) {
    if (!(scores[i] >= 0.0)) return fail(ORC_USAGE, "negative leverage score");
    total += scores[i];
  }
  if (total == 0.0) return fail(ORC_NUMERICAL, "zero score sum; distribution undefined");
  for (int64_t i = 0; i < w; ++i) out[i] = scores[i] / total;
  return ORC_OK;
}

/* ======================================================================
 * sketch.cpp:20-59 -- inverse-CDF sampling with replacement
 * ==================================================================== */
int orc_sample_rows(const double* pi, int64_t n, int64_t c, uint64_t seed, int64_t* idx,
                    double* weights) {
  if (n < 1) return fail(ORC_DATA, "empty distribution");
  if (c < 1) return fail(ORC_USAGE, "sample count must be positive");
  double total = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    if (!(pi[i] >= 0.0)) return fail(ORC_DATA, "distribution has a negative entry");
    total += pi[i];
  }
  if (fabs(total - 1.0) > 1e-8) return fail(ORC_DATA, "distribution sums to %g, not 1", total);
  double* cdf = XMALLOC(double, n);
  double acc = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    acc += pi[i];
    cdf[i] = acc;
  }
  cdf[n - 1] = acc;
  orc_rng rng;
  orc_rng_init(&rng, seed);
  const double cd = (double)c;
  for (int64_t t = 0; t < c; ++t) {
    const double u = orc_rng_uniform01(&rng) * acc;
    /* std::upper_bound: first element > u */
    int64_t lo = 0, hi = n;
    while (lo < hi) {
      const int64_t mid = lo + (hi - lo) / 2;
      if (u < cdf[mid])
        hi = mid;
      else
        lo = mid + 1;
    }
    int64_t i = lo;
    if (i == n) --i;
    while (pi[i] == 0.0 && i + 1 < n) ++i;
    while (pi[i] == 0.0 && i > 0) --i;
    idx[t] = i;
    weights[t] = 1.0 / sqrt(cd * pi[i] / total);
  }
  free(cdf);
  return ORC_OK;
}

/* sketch.cpp:61-79 for the implicit window system (y, n_used, p) */
int orc_apply_sample(const double* y, int64_t n_used, int p, const int64_t* idx,
                     const double* weights, int64_t c, int width, double* a_out, double* b_out) {
  if (width < 1 || width > p) return fail(ORC_USAGE, "invalid column width");
  const int64_t rows = n_used - p;
  for (int64_t t = 0; t < c; ++t) {
    const int64_t i = idx[t];
    if (i < 0 || i >= rows) return fail(ORC_USAGE, "sample index out of range");
    const double w = weights[t];
    for (int j = 0; j < width; ++j) a_out[t + (int64_t)j * c] = w * y[p + i - 1 - j];
    b_out[t] = w * y[p + i];
  }
  return ORC_OK;
}

/* ======================================================================
 * Column-pivoting Householder QR -- restates Eigen's ColPivHouseholderQR
 * (used at toeplitz.cpp:61-71, 108-114; repeated_halving.cpp:58-64):
 * greedy max-updated-norm pivot, LAPACK-style norm downdate (lawn176),
 * nonzero-pivot tracking, rank = #{|r_ii| > threshold * max|r_ii|}.
 * ==================================================================== */
typedef struct {
  int64_t rows, cols, size;
  double* qr;     /* col-major rows x cols */
  double* hc;     /* [size] */
  int64_t* perm;  /* perm[i] = original column at position i */
  int64_t nzp;
  double maxpivot;
} cpqr_t;

static void cpqr_free(cpqr_t* f) {
  free(f->qr);
  free(f->hc);
  free(f->perm);
}

static void cpqr_compute(cpqr_t* f, const double* a, int64_t rows, int64_t cols) {
  f->rows = rows;
  f->cols = cols;
  f->size = rows < cols ? rows : cols;
  f->qr = XMALLOC(double, rows * cols);
  memcpy(f->qr, a, sizeof(double) * (size_t)(rows * cols));
  f->hc = XMALLOC(double, f->size);
  f->perm = XMALLOC(int64_t, cols);
  double* upd = XMALLOC(double, cols);
  double* dir = XMALLOC(double, cols);
  double* q = f->qr;
  double maxnorm = 0.0;
  for (int64_t k = 0; k < cols; ++k) {
    f->perm[k] = k;
    dir[k] = sqrt(sqnorm(q + k * rows, rows));
    upd[k] = dir[k];
    if (upd[k] > maxnorm) maxnorm = upd[k];
  }
  const double th_help = (maxnorm * DBL_EPSILON) * (maxnorm * DBL_EPSILON) / (double)rows;
  const double downdate_th = sqrt(DBL_EPSILON);
  f->nzp = f->size;
  f->maxpivot = 0.0;
  for (int64_t k = 0; k < f->size; ++k) {
    int64_t big = k;
    for (int64_t j = k + 1; j < cols; ++j)
      if (upd[j] > upd[big]) big = j;
    const double big_sq = upd[big] * upd[big];
    if (f->nzp == f->size && big_sq < th_help * (double)(rows - k)) f->nzp = k;
    if (big != k) {
      double* ck = q + k * rows;
      double* cb = q + big * rows;
      for (int64_t i = 0; i < rows; ++i) {
        const double t = ck[i];
        ck[i] = cb[i];
        cb[i] = t;
      }
      double t = upd[k]; upd[k] = upd[big]; upd[big] = t;
      t = dir[k]; dir[k] = dir[big]; dir[big] = t;
      const int64_t ti = f->perm[k]; f->perm[k] = f->perm[big]; f->perm[big] = ti;
    }
    /* makeHouseholderInPlace on column k, rows k.. */
    double* x = q + k * rows + k;
    const int64_t len = rows - k;
    const double c0 = x[0];
    const double tail_sq = len == 1 ? 0.0 : sqnorm(x + 1, len - 1);
    double tau, beta;
    if (tail_sq <= DBL_MIN) {
      tau = 0.0;
      beta = c0;
      for (int64_t i = 1; i < len; ++i) x[i] = 0.0;
    } else {
      beta = sqrt(c0 * c0 + tail_sq);
      if (c0 >= 0.0) beta = -beta;
      const double d = c0 - beta;
      for (int64_t i = 1; i < len; ++i) x[i] = x[i] / d;
      tau = (beta - c0) / beta;
    }
    x[0] = beta;
    f->hc[k] = tau;
    if (fabs(beta) > f->maxpivot) f->maxpivot = fabs(beta);
    /* applyHouseholderOnTheLeft on bottomRightCorner(rows-k, cols-k-1)
     * (columns independent: thread count does not change the result) */
#pragma omp parallel for schedule(static) if ((cols - k) * len > 65536)
    for (int64_t j = k + 1; j < cols; ++j) {
      double* cj = q + j * rows + k;
      if (len == 1) {
        cj[0] *= (1.0 - tau);
      } else if (tau != 0.0) {
        const double tmp = dot(x + 1, cj + 1, len - 1) + cj[0];
        cj[0] -= tau * tmp;
        axpy(-tau * tmp, x + 1, cj + 1, len - 1);
      }
    }
    /* norm downdate */
#pragma omp parallel for schedule(static) if ((cols - k) * len > 65536)
    for (int64_t j = k + 1; j < cols; ++j) {
      if (upd[j] != 0.0) {
        double temp = fabs(q[j * rows + k]) / upd[j];
        temp = (1.0 + temp) * (1.0 - temp);
        if (temp < 0.0) temp = 0.0;
        const double ratio = upd[j] / dir[j];
        const double temp2 = temp * ratio * ratio;
        if (temp2 <= downdate_th) {
          dir[j] = sqrt(sqnorm(q + j * rows + k + 1, rows - k - 1));
          upd[j] = dir[j];
        } else {
          upd[j] *= sqrt(temp);
        }
      }
    }
  }
  free(upd);
  free(dir);
}

static int64_t cpqr_rank(const cpqr_t* f, double threshold) {
  const double pre = fabs(f->maxpivot) * threshold;
  int64_t r = 0;
  for (int64_t i = 0; i < f->nzp; ++i) r += fabs(f->qr[i * f->rows + i]) > pre;
  return r;
}

/* Apply H_k (k = 0..len-1 in order) to vector c (length rows): Q^T c. */
static void cpqr_apply_qt(const cpqr_t* f, int64_t nh, double* c) {
  const int64_t rows = f->rows;
  for (int64_t k = 0; k < nh; ++k) {
    const double tau = f->hc[k];
    const int64_t len = rows - k;
    const double* v = f->qr + k * rows + k;
    if (len == 1) {
      c[k] *= (1.0 - tau);
    } else if (tau != 0.0) {
      const double tmp = dot(v + 1, c + k + 1, len - 1) + c[k];
      c[k] -= tau * tmp;
      axpy(-tau * tmp, v + 1, c + k + 1, len - 1);
    }
  }
}

/* Apply Q = H_0 ... H_{nh-1} to vector c (H_{nh-1} first). */
static void cpqr_apply_q(const cpqr_t* f, int64_t nh, double* c) {
  const int64_t rows = f->rows;
  for (int64_t k = nh - 1; k >= 0; --k) {
    const double tau = f->hc[k];
    const int64_t len = rows - k;
    const double* v = f->qr + k * rows + k;
    if (len == 1) {
      c[k] *= (1.0 - tau);
    } else if (tau != 0.0) {
      const double tmp = dot(v + 1, c + k + 1, len - 1) + c[k];
      c[k] -= tau * tmp;
      axpy(-tau * tmp, v + 1, c + k + 1, len - 1);
    }
  }
}

/* Eigen ColPivHouseholderQR::_solve_impl for the full-rank case */
static void cpqr_solve(const cpqr_t* f, const double* b, double* x) {
  const int64_t rows = f->rows, n = f->nzp;
  double* c = XMALLOC(double, rows);
  memcpy(c, b, sizeof(double) * (size_t)rows);
  cpqr_apply_qt(f, n, c);
  for (int64_t i = n - 1; i >= 0; --i) {
    double s = c[i];
    for (int64_t j = i + 1; j < n; ++j) s -= f->qr[j * rows + i] * c[j];
    c[i] = s / f->qr[i * rows + i];
  }
  for (int64_t i = 0; i < f->cols; ++i) x[i] = 0.0;
  for (int64_t i = 0; i < n; ++i) x[f->perm[i]] = c[i];
  free(c);
}

/* ======================================================================
 * Minimum-norm least squares via one-sided Jacobi SVD (stands in for
 * Eigen's BDCSVD at toeplitz.cpp:75-81; same rank rule: singular values
 * below max(rows,cols)*eps*sigma_max are dropped).
 * ==================================================================== */
/* one-sided Jacobi on M (m x n, col-major, m >= n); V (n x n) accumulates.
 * Round-robin (tournament) pair order: the n/2 pairs of a round touch
 * disjoint columns, so a round runs in parallel and the result does not
 * depend on the thread count. */
static void jacobi_svd(double* M, int64_t m, int64_t n, double* V, double* sigma) {
  for (int64_t i = 0; i < n * n; ++i) V[i] = 0.0;
  for (int64_t i = 0; i < n; ++i) V[i * n + i] = 1.0;
  const int64_t np2 = n + (n & 1); /* players; index n is a bye when n is odd */
  for (int sweep = 0; sweep < 80 && n > 1; ++sweep) {
    int rotated = 0;
    for (int64_t rd = 0; rd < np2 - 1; ++rd) {
#pragma omp parallel for schedule(static) reduction(| : rotated) if (m * n > 40000)
      for (int64_t t = 0; t < np2 / 2; ++t) {
        int64_t a = (rd + t) % (np2 - 1);
        int64_t b = t == 0 ? np2 - 1 : (rd - t + (np2 - 1)) % (np2 - 1);
        if (a >= n || b >= n) continue;
        const int64_t i = a < b ? a : b, j = a < b ? b : a;
        double* mi = M + i * m;
        double* mj = M + j * m;
        const double alpha = sqnorm(mi, m), beta = sqnorm(mj, m), gamma = dot(mi, mj, m);
        if (gamma == 0.0 || fabs(gamma) <= DBL_EPSILON * sqrt(alpha * beta)) continue;
        rotated = 1;
        const double zeta = (beta - alpha) / (2.0 * gamma);
        const double tt = (zeta >= 0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        const double cs = 1.0 / sqrt(1.0 + tt * tt), sn = cs * tt;
        for (int64_t r = 0; r < m; ++r) {
          const double x = mi[r], y = mj[r];
          mi[r] = cs * x - sn * y;
          mj[r] = sn * x + cs * y;
        }
        double* vi = V + i * n;
        double* vj = V + j * n;
        for (int64_t r = 0; r < n; ++r) {
          const double x = vi[r], y = vj[r];
          vi[r] = cs * x - sn * y;
          vj[r] = sn * x + cs * y;
        }
      }
    }
    if (!rotated) break;
  }
  for (int64_t i = 0; i < n; ++i) sigma[i] = sqrt(sqnorm(M + i * m, m));
}

static void minnorm_solve(const double* a, int64_t rows, int64_t cols, const double* b,
                          double* x, double tol) {
  for (int64_t i = 0; i < cols; ++i) x[i] = 0.0;
  if (rows >= cols) {
    /* R = upper-triangular factor of an unpivoted Householder QR; c = Q^T b */
    cpqr_t f;
    f.rows = rows; f.cols = cols; f.size = cols;
    f.qr = XMALLOC(double, rows * cols);
    memcpy(f.qr, a, sizeof(double) * (size_t)(rows * cols));
    f.hc = XMALLOC(double, cols);
    f.perm = NULL;
    for (int64_t k = 0; k < cols; ++k) {
      double* xk = f.qr + k * rows + k;
      const int64_t len = rows - k;
      const double c0 = xk[0];
      const double tail_sq = len == 1 ? 0.0 : sqnorm(xk + 1, len - 1);
      double tau, beta;
      if (tail_sq <= DBL_MIN) {
        tau = 0.0; beta = c0;
        for (int64_t i = 1; i < len; ++i) xk[i] = 0.0;
      } else {
        beta = sqrt(c0 * c0 + tail_sq);
        if (c0 >= 0.0) beta = -beta;
        const double d = c0 - beta;
        for (int64_t i = 1; i < len; ++i) xk[i] /= d;
        tau = (beta - c0) / beta;
      }
      xk[0] = beta;
      f.hc[k] = tau;
#pragma omp parallel for schedule(static) if ((cols - k) * len > 65536)
      for (int64_t j = k + 1; j < cols; ++j) {
        double* cj = f.qr + j * rows + k;
        if (len == 1) cj[0] *= (1.0 - tau);
        else if (tau != 0.0) {
          const double tmp = dot(xk + 1, cj + 1, len - 1) + cj[0];
          cj[0] -= tau * tmp;
          axpy(-tau * tmp, xk + 1, cj + 1, len - 1);
        }
      }
    }
    double* c = XMALLOC(double, rows);
    memcpy(c, b, sizeof(double) * (size_t)rows);
    cpqr_apply_qt(&f, cols, c);
    double* R = XMALLOC(double, cols * cols);
    for (int64_t j = 0; j < cols; ++j)
      for (int64_t i = 0; i < cols; ++i) R[j * cols + i] = i <= j ? f.qr[j * rows + i] : 0.0;
    double* V = XMALLOC(double, cols * cols);
    double* s = XMALLOC(double, cols);
    jacobi_svd(R, cols, cols, V, s); /* R overwritten by U*Sigma */
    double smax = 0.0;
    for (int64_t i = 0; i < cols; ++i) if (s[i] > smax) smax = s[i];
    double pre = smax * tol;
    if (pre < DBL_MIN) pre = DBL_MIN;
    for (int64_t i = 0; i < cols; ++i) {
      if (!(s[i] >= pre)) continue;
      /* (u_i^T c)/s_i with u_i = R_col_i / s_i */
      const double coef = dot(R + i * cols, c, cols) / (s[i] * s[i]);
      axpy(coef, V + i * cols, x, cols);
    }
    free(c); free(R); free(V); free(s); free(f.qr); free(f.hc);
  } else {
    /* M = A^T (cols x rows); A^T = U S W^T, x = U S^+ W^T b */
    double* M = XMALLOC(double, cols * rows);
    for (int64_t i = 0; i < rows; ++i)
      for (int64_t j = 0; j < cols; ++j) M[i * cols + j] = a[j * rows + i];
    double* W = XMALLOC(double, rows * rows);
    double* s = XMALLOC(double, rows);
    jacobi_svd(M, cols, rows, W, s);
    double smax = 0.0;
    for (int64_t i = 0; i < rows; ++i) if (s[i] > smax) smax = s[i];
    double pre = smax * tol;
    if (pre < DBL_MIN) pre = DBL_MIN;
    for (int64_t i = 0; i < rows; ++i) {
      if (!(s[i] >= pre)) continue;
      const double coef = dot(W + i * rows, b, rows) / (s[i] * s[i]);
      axpy(coef, M + i * cols, x, cols);
    }
    free(M); free(W); free(s);
  }
}

/* ||A x - b|| of a column-major system evaluated in double-double (exact
 * products by fma, TwoSum accumulation): the residual of a given x, free of
 * the cancellation that swamps a plain fp64 evaluation when ||r|| << ||b||
 * (C4-like series, |y| ~ 1e19 against unit innovations).  Test helper. */
static inline void dd_acc_c(double* h, double* l, double a, double b) {
  const double p = a * b;
  const double e = fma(a, b, -p);
  const double s = *h + p;
  const double bb = s - *h;
  *l += ((*h - (s - bb)) + (p - bb)) + e;
  *h = s;
}
double orc_residual_norm_dd(const double* a, int64_t rows, int64_t cols, const double* b, const double* x) {
  double th = 0.0, tl = 0.0;
  for (int64_t i = 0; i < rows; ++i) {
    double h = 0.0, l = 0.0;
    for (int64_t j = 0; j < cols; ++j) dd_acc_c(&h, &l, a[i + j * rows], x[j]);
    dd_acc_c(&h, &l, b[i], -1.0);
    const double r = h + l;
    dd_acc_c(&th, &tl, r, r);
  }
  return sqrt(th + tl);
}

/* toeplitz.cpp:57-85 */
int orc_solve_exact(const double* a, int64_t rows, int64_t cols, const double* b, double* x,
                    int* method_out, int64_t* rank_out) {
  if (rows == 0 || cols == 0) return fail(ORC_USAGE, "empty system");
  const double tol = (double)(rows > cols ? rows : cols) * DBL_EPSILON;
  int solved = 0;
  if (rows >= cols) {
    cpqr_t f;
    cpqr_compute(&f, a, rows, cols);
    const int64_t rank = cpqr_rank(&f, tol);
    if (rank_out) *rank_out = rank;
    if (rank == cols) {
      cpqr_solve(&f, b, x);
      if (method_out) *method_out = ORC_SOLVE_QR;
      solved = 1;
    }
    cpqr_free(&f);
  } else if (rank_out) {
    *rank_out = -1;
  }
  if (!solved) {
    minnorm_solve(a, rows, cols, b, x, tol);
    if (method_out) *method_out = ORC_SOLVE_SVD;
  }
  return ORC_OK;
}

/* toeplitz.cpp:100-115 */
int orc_exact_leverage(const double* a, int64_t rows, int64_t cols, double* out) {
  if (rows < cols) return fail(ORC_USAGE, "leverage scores need rows >= cols");
  if (cols == 0) return fail(ORC_USAGE, "empty matrix");
  cpqr_t f;
  cpqr_compute(&f, a, rows, cols);
  const double tol = (double)(rows > cols ? rows : cols) * DBL_EPSILON;
  if (cpqr_rank(&f, tol) != cols) {
    cpqr_free(&f);
    return fail(ORC_NUMERICAL, "matrix is rank deficient; leverage scores undefined");
  }
  for (int64_t i = 0; i < rows; ++i) out[i] = 0.0;
  double* e = XMALLOC(double, rows);
  for (int64_t j = 0; j < cols; ++j) {
    for (int64_t i = 0; i < rows; ++i) e[i] = i == j ? 1.0 : 0.0;
    cpqr_apply_q(&f, f.size, e);
    for (int64_t i = 0; i < rows; ++i) out[i] += e[i] * e[i];
  }
  free(e);
  cpqr_free(&f);
  return ORC_OK;
}

/* sketch.cpp:241-253 -- G (g x rows) drawn column by column of G */
int orc_gaussian_apply(int64_t g, uint64_t seed, const double* m, int64_t rows, int64_t cols,
                       double* out) {
  if (g < 1) return fail(ORC_USAGE, "sketch needs at least one row");
  for (int64_t i = 0; i < g * cols; ++i) out[i] = 0.0;
  /* the normals in stream order (column j of G = draws j*g .. j*g+g-1), then
   * every output column accumulates over j in order (columns in parallel) */
  double* G = XMALLOC(double, g * rows);
  orc_rng rng;
  orc_rng_init(&rng, seed);
  for (int64_t j = 0; j < rows; ++j)
    for (int64_t i = 0; i < g; ++i) G[j * g + i] = orc_rng_normal(&rng);
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t l = 0; l < cols; ++l) {
    double* o = out + l * g;
    for (int64_t j = 0; j < rows; ++j) {
      const double mv = m[l * rows + j];
      const double* col = G + j * g;
      for (int64_t i = 0; i < g; ++i) o[i] += col[i] * mv;
    }
  }
  free(G);
  return ORC_OK;
}

/* toeplitz.cpp:133-138 */
int orc_select_order(const double* taus, int p_bar, double bound) {
  for (int h = p_bar; h >= 1; --h)
    if (fabs(taus[h - 1]) >= bound) return h;
  return 0;
}

/* ======================================================================
 * lsar.cpp:55-124 -- LsarDriver + lsar_fit
 * ==================================================================== */
static int lsar_solve_at(const double* y, int64_t w, int p, int64_t c, uint64_t seed,
                         const double* scores, const int64_t* fidx, const double* fw,
                         int64_t* idx, double* wt, double* dist, double* a, double* b,
                         double* phi, double* r, int* method) {
  int st;
  const int64_t n_used = w + p;
  if (fidx) {
    memcpy(idx, fidx, sizeof(int64_t) * (size_t)c);
    memcpy(wt, fw, sizeof(double) * (size_t)c);
  } else {
    if ((st = orc_leverage_to_distribution(scores, w, dist))) return st;
    if ((st = orc_sample_rows(dist, w, c, orc_derive_seed(seed, (uint64_t)p), idx, wt)))
      return st;
  }
  if ((st = orc_apply_sample(y, n_used, p, idx, wt, c, p, a, b))) return st;
  if ((st = orc_solve_exact(a, c, p, b, phi, method, NULL))) return st;
  return orc_residuals(y, n_used, p, phi, r);
}

int orc_lsar_fit(const double* y, int64_t n, int p_bar, int64_t c, uint64_t seed,
                 orc_lsar_diag* diag, double* taus, double* coefs_packed, double* lag_seconds,
                 int* p_star) {
  if (p_bar < 1) return fail(ORC_USAGE, "maximum lag must be at least 1");
  if (n <= (int64_t)p_bar + 1) return fail(ORC_DATA, "series too short for maximum lag %d", p_bar);
  if (c < p_bar) return fail(ORC_USAGE, "sample count below maximum lag");
  const int64_t w = n - p_bar;
  double* s = XMALLOC(double, w);
  double* s2 = XMALLOC(double, w);
  double* r = XMALLOC(double, w);
  double* dist = XMALLOC(double, w);
  double* a = XMALLOC(double, c * (int64_t)p_bar);
  double* b = XMALLOC(double, c);
  int64_t* idx = XMALLOC(int64_t, c);
  double* wt = XMALLOC(double, c);
  double* phi = XMALLOC(double, p_bar);
  int st = ORC_OK;
  int64_t off = 0;
  for (int p = 1; p <= p_bar; ++p) {
    const double t0 = now_seconds();
    if (p == 1) {
      st = orc_init_leverage_p1(y, w, s);
    } else {
      st = orc_leverage_update(s, r, w, s2);
      if (!st) { double* t = s; s = s2; s2 = t; }
    }
    if (st) break;
    const int64_t* fi = diag && diag->fixed_idx ? diag->fixed_idx + (int64_t)(p - 1) * c : NULL;
    const double* fw = diag && diag->fixed_w ? diag->fixed_w + (int64_t)(p - 1) * c : NULL;
    int method = 0;
    st = lsar_solve_at(y, w, p, c, seed, s, fi, fw, idx, wt, dist, a, b, phi, r, &method);
    if (st) break;
    if (lag_seconds) lag_seconds[p - 1] = now_seconds() - t0;
    taus[p - 1] = phi[p - 1];
    if (coefs_packed) memcpy(coefs_packed + off, phi, sizeof(double) * (size_t)p);
    off += p;
    if (diag) {
      if (diag->idx_out) memcpy(diag->idx_out + (int64_t)(p - 1) * c, idx, sizeof(int64_t) * (size_t)c);
      if (diag->w_out) memcpy(diag->w_out + (int64_t)(p - 1) * c, wt, sizeof(double) * (size_t)c);
      if (diag->rnorm2_out) diag->rnorm2_out[p - 1] = seq_sqnorm(r, w);
      if (diag->ssum_out) {
        double ss = 0.0;
        for (int64_t i = 0; i < w; ++i) ss += s[i];
        diag->ssum_out[p - 1] = ss;
      }
      if (diag->scores_all) memcpy(diag->scores_all + (int64_t)(p - 1) * w, s, sizeof(double) * (size_t)w);
      if (diag->method_out) diag->method_out[p - 1] = method;
      if (p == p_bar) {
        if (diag->scores_out) memcpy(diag->scores_out, s, sizeof(double) * (size_t)w);
        if (diag->resid_out) memcpy(diag->resid_out, r, sizeof(double) * (size_t)w);
      }
    }
  }
  if (!st && p_star) *p_star = orc_select_order(taus, p_bar, 1.96 / sqrt((double)c));
  free(s); free(s2); free(r); free(dist); free(a); free(b); free(idx); free(wt); free(phi);
  return st;
}

/* lsar_fit's recursion and draws replayed from given per-lag coefficients
 * (the solve skipped): with the coefficients orc_lsar_fit produced, every
 * score, residual and draw is bit-identical to that run (same functions,
 * same order).  Lets a test reproduce the oracle's samples of a BASELINE-size
 * fit from a small fixture (the packed coefficients) in O(p_bar n) time. */
int orc_lsar_replay(const double* y, int64_t n, int p_bar, int64_t c, uint64_t seed,
                    const double* coefs_packed, int64_t* idx_out, double* w_out, double* rnorm2_out,
                    double* ssum_out) {
  if (p_bar < 1) return fail(ORC_USAGE, "maximum lag must be at least 1");
  if (n <= (int64_t)p_bar + 1) return fail(ORC_DATA, "series too short for maximum lag %d", p_bar);
  if (c < p_bar) return fail(ORC_USAGE, "sample count below maximum lag");
  const int64_t w = n - p_bar;
  double* s = XMALLOC(double, w);
  double* s2 = XMALLOC(double, w);
  double* r = XMALLOC(double, w);
  double* dist = XMALLOC(double, w);
  int st = ORC_OK;
  int64_t off = 0;
  for (int p = 1; p <= p_bar && !st; ++p) {
    if (p == 1) {
      st = orc_init_leverage_p1(y, w, s);
    } else {
      st = orc_leverage_update(s, r, w, s2);
      if (!st) { double* t = s; s = s2; s2 = t; }
    }
    if (st) break;
    st = orc_leverage_to_distribution(s, w, dist);
    if (!st)
      st = orc_sample_rows(dist, w, c, orc_derive_seed(seed, (uint64_t)p), idx_out + (int64_t)(p - 1) * c,
                           w_out + (int64_t)(p - 1) * c);
    if (!st) st = orc_residuals(y, w + p, p, coefs_packed + off, r);
    off += p;
    if (st) break;
    if (rnorm2_out) rnorm2_out[p - 1] = seq_sqnorm(r, w);
    if (ssum_out) {
      double ss = 0.0;
      for (int64_t i = 0; i < w; ++i) ss += s[i];
      ssum_out[p - 1] = ss;
    }
  }
  free(s); free(s2); free(r); free(dist);
  return st;
}

double orc_lsar_time_one_lag(const double* y, int64_t n, int p_bar, int64_t c, int p,
                             uint64_t seed) {
  if (p < 1 || p > p_bar || n <= (int64_t)p_bar + 1 || c < p_bar) return -1.0;
  const int64_t w = n - p_bar;
  double* s = XMALLOC(double, w);
  double* s2 = XMALLOC(double, w);
  double* r = XMALLOC(double, w);
  double* dist = XMALLOC(double, w);
  double* a = XMALLOC(double, c * (int64_t)p);
  double* b = XMALLOC(double, c);
  int64_t* idx = XMALLOC(int64_t, c);
  double* wt = XMALLOC(double, c);
  double* phi = XMALLOC(double, p);
  /* stand-in state: s_{p-1} from the lag-1 closed form, r_{p-1} = -y */
  orc_init_leverage_p1(y, w, s);
  for (int64_t i = 0; i < w; ++i) r[i] = -y[i];
  int method;
  const double t0 = now_seconds();
  int st = p == 1 ? ORC_OK : orc_leverage_update(s, r, w, s2);
  if (!st)
    st = lsar_solve_at(y, w, p, c, seed, p == 1 ? s : s2, NULL, NULL, idx, wt, dist, a, b, phi,
                       r, &method);
  const double dt = now_seconds() - t0;
  free(s); free(s2); free(r); free(dist); free(a); free(b); free(idx); free(wt); free(phi);
  return st ? -1.0 : dt;
}

/* ======================================================================
 * repeated_halving.cpp
 * ==================================================================== */
int64_t orc_default_base_threshold(int64_t c, int64_t k) { /* repeated_halving.hpp:67-70 */
  const int64_t logk = (int64_t)ceil(log((double)k + 1.0));
  const int64_t v = 10 * k * logk;
  return c > v ? c : v;
}

int64_t orc_default_gaussian_rows(int64_t n) { /* sketch.hpp:42-44 */
  return (int64_t)ceil(8.0 * log((double)n));
}

void orc_rh_defaults(int64_t n, int64_t k, int64_t c, uint64_t seed, orc_rh_cfg* out) {
  /* repeated_halving.cpp:33-41 */
  out->sample_count = c;
  out->base_threshold = orc_default_base_threshold(c, k);
  out->gaussian_rows = orc_default_gaussian_rows(n > 2 ? n : 2);
  out->seed = seed;
}

/* LeverageKernel (repeated_halving.cpp:54-90) */
typedef struct {
  int64_t k;
  double* r;      /* k x k col-major upper */
  int64_t* perm;
  double* mix;    /* g x k col-major, or NULL */
  int64_t g;
} levker_t;

static int levker_init(levker_t* L, const double* bm, int64_t brows, int64_t k, int64_t g,
                       uint64_t seed) {
  memset(L, 0, sizeof *L);
  if (brows < k) return fail(ORC_NUMERICAL, "reference matrix has too few rows");
  cpqr_t f;
  cpqr_compute(&f, bm, brows, k);
  const double tol = (double)(brows > k ? brows : k) * DBL_EPSILON;
  if (cpqr_rank(&f, tol) != k) {
    cpqr_free(&f);
    return fail(ORC_NUMERICAL, "reference matrix is rank deficient");
  }
  L->k = k;
  L->r = XMALLOC(double, k * k);
  for (int64_t j = 0; j < k; ++j)
    for (int64_t i = 0; i < k; ++i) L->r[j * k + i] = i <= j ? f.qr[j * brows + i] : 0.0;
  L->perm = XMALLOC(int64_t, k);
  memcpy(L->perm, f.perm, sizeof(int64_t) * (size_t)k);
  if (g > 0) {
    double* thin = XMALLOC(double, brows * k);
    for (int64_t j = 0; j < k; ++j) {
      double* e = thin + j * brows;
      for (int64_t i = 0; i < brows; ++i) e[i] = i == j ? 1.0 : 0.0;
      cpqr_apply_q(&f, f.size, e);
    }
    L->mix = XMALLOC(double, g * k);
    orc_gaussian_apply(g, seed, thin, brows, k, L->mix);
    const double sg = sqrt((double)g);
    for (int64_t i = 0; i < g * k; ++i) L->mix[i] /= sg;
    L->g = g;
    free(thin);
  }
  cpqr_free(&f);
  return ORC_OK;
}

static void levker_free(levker_t* L) {
  free(L->r);
  free(L->perm);
  free(L->mix);
}

/* score of one row x (length k) */
static double levker_score(const levker_t* L, const double* x, double* z) {
  const int64_t k = L->k;
  for (int64_t i = 0; i < k; ++i) z[i] = x[L->perm[i]];
  /* R^T z' = z (forward substitution) */
  for (int64_t i = 0; i < k; ++i) {
    double s = z[i];
    for (int64_t l = 0; l < i; ++l) s -= L->r[i * k + l] * z[l];
    z[i] = s / L->r[i * k + i];
  }
  double out = 0.0;
  if (L->mix) {
    for (int64_t gi = 0; gi < L->g; ++gi) {
      double acc = 0.0;
      for (int64_t j = 0; j < k; ++j) acc += L->mix[j * L->g + gi] * z[j];
      out += acc * acc;
    }
  } else {
    for (int64_t j = 0; j < k; ++j) out += z[j] * z[j];
  }
  return out;
}

int orc_generalized_leverage(const double* cm, int64_t rows, const double* b, int64_t brows,
                             int64_t k, int64_t sketch_rows, uint64_t sketch_seed, double* out) {
  levker_t L;
  int st = levker_init(&L, b, brows, k, sketch_rows > 0 ? sketch_rows : 0, sketch_seed);
  if (st) return st;
  double* x = XMALLOC(double, k);
  double* z = XMALLOC(double, k);
  for (int64_t i = 0; i < rows; ++i) {
    for (int64_t j = 0; j < k; ++j) x[j] = cm[j * rows + i];
    out[i] = levker_score(&L, x, z);
  }
  free(x); free(z);
  levker_free(&L);
  return ORC_OK;
}

/* AugmentedRowSource::gather (repeated_halving.cpp:22-31) for the full
 * lag-p_bar system: row i = (y[p+i-1], ..., y[i], y[p+i]). */
static void aug_row(const double* y, int p, int64_t i, double* out) {
  for (int j = 0; j < p; ++j) out[j] = y[p + i - 1 - j];
  out[p] = y[p + i];
}

static int rh_fit_impl(const double* y, int64_t n, int p_bar, int64_t c, const orc_rh_cfg* cfg_in,
                       uint64_t seed, orc_rh_diag* diag, double* taus, double* coefs_packed,
                       double* lag_seconds, double* upfront_seconds, int* p_star,
                       int upfront_only) {
  /* repeated_halving.cpp:191-232 */
  if (p_bar < 1) return fail(ORC_USAGE, "maximum lag must be at least 1");
  if (n <= (int64_t)p_bar + 1) return fail(ORC_DATA, "series too short for maximum lag %d", p_bar);
  if (c < p_bar) return fail(ORC_USAGE, "sample count below maximum lag");
  const int64_t m = n - p_bar;
  const int64_t k = p_bar + 1;
  orc_rh_cfg cfg;
  if (cfg_in) cfg = *cfg_in;
  else orc_rh_defaults(m, k, c, orc_derive_seed(seed, 0x5c07e5u), &cfg);
  /* RHConfig::validate (repeated_halving.cpp:43-47) */
  if (cfg.sample_count < 1) return fail(ORC_USAGE, "sample count must be positive");
  if (cfg.base_threshold < cfg.sample_count) return fail(ORC_USAGE, "base threshold below sample count");
  if (cfg.gaussian_rows < 1) return fail(ORC_USAGE, "need at least one sketch row");

  int st = ORC_OK;
  double t0 = now_seconds();
  /* ---- repeated_halving (repeated_halving.cpp:126-180) ---- */
  int64_t* lvl_ptr[64];
  int64_t lvl_size[64];
  int nlev = 1;
  lvl_ptr[0] = XMALLOC(int64_t, m);
  for (int64_t i = 0; i < m; ++i) lvl_ptr[0][i] = i;
  lvl_size[0] = m;
  while (lvl_size[nlev - 1] > cfg.base_threshold) {
    const int64_t size = lvl_size[nlev - 1];
    const int64_t half = size / 2;
    int64_t* next = XMALLOC(int64_t, size);
    memcpy(next, lvl_ptr[nlev - 1], sizeof(int64_t) * (size_t)size);
    orc_rng rng;
    orc_rng_init(&rng, orc_derive_seed(cfg.seed, 0x10000u + (uint64_t)nlev));
    for (int64_t i = 0; i < half; ++i) {
      const int64_t j = i + (int64_t)orc_rng_below(&rng, (uint64_t)(size - i));
      const int64_t t = next[i]; next[i] = next[j]; next[j] = t;
    }
    qsort(next, (size_t)half, sizeof(int64_t), cmp_i64);
    lvl_ptr[nlev] = next;
    lvl_size[nlev] = half;
    ++nlev;
  }
  const int depth = nlev - 1;
  int64_t arows = lvl_size[depth];
  double* approx = XMALLOC(double, arows * k);
  double* row = XMALLOC(double, k);
  double* z = XMALLOC(double, k);
  for (int64_t t = 0; t < arows; ++t) {
    aug_row(y, p_bar, lvl_ptr[depth][t], row);
    for (int64_t j = 0; j < k; ++j) approx[j * arows + t] = row[j];
  }
  const int64_t sc = cfg.sample_count;
  int64_t* sidx = XMALLOC(int64_t, sc);
  double* sw = XMALLOC(double, sc);
  for (int i = depth - 1; i >= 0 && !st; --i) {
    const int64_t len = lvl_size[i];
    const int64_t* cur = lvl_ptr[i];
    levker_t L;
    st = levker_init(&L, approx, arows, k, cfg.gaussian_rows,
                     orc_derive_seed(cfg.seed, 0x20000u + (unsigned)i));
    if (st) break;
    double* sco = XMALLOC(double, len);
#pragma omp parallel
    {
      double* prow = XMALLOC(double, k);
      double* pz = XMALLOC(double, k);
#pragma omp for schedule(static)
      for (int64_t t = 0; t < len; ++t) {
        aug_row(y, p_bar, cur[t], prow);
        sco[t] = levker_score(&L, prow, pz);
      }
      free(prow); free(pz);
    }
    levker_free(&L);
    st = orc_leverage_to_distribution(sco, len, sco);
    if (!st)
      st = orc_sample_rows(sco, len, sc, orc_derive_seed(cfg.seed, 0x30000u + (unsigned)i), sidx, sw);
    free(sco);
    if (st) break;
    if (diag && diag->up_idx) memcpy(diag->up_idx + (int64_t)i * sc, sidx, sizeof(int64_t) * (size_t)sc);
    if (diag && diag->up_w) memcpy(diag->up_w + (int64_t)i * sc, sw, sizeof(double) * (size_t)sc);
    double* nxt = XMALLOC(double, sc * k);
    for (int64_t t = 0; t < sc; ++t) {
      aug_row(y, p_bar, cur[sidx[t]], row);
      for (int64_t j = 0; j < k; ++j) nxt[j * sc + t] = row[j] * sw[t];
    }
    free(approx);
    approx = nxt;
    arows = sc;
  }
  double* scores = NULL;
  if (!st) {
    /* rh_leverage_scores: final unsketched pass (repeated_halving.cpp:182-189) */
    levker_t L;
    st = levker_init(&L, approx, arows, k, 0, 0);
    if (!st) {
      scores = XMALLOC(double, m);
#pragma omp parallel
      {
        double* prow = XMALLOC(double, k);
        double* pz = XMALLOC(double, k);
#pragma omp for schedule(static)
        for (int64_t i = 0; i < m; ++i) {
          aug_row(y, p_bar, i, prow);
          scores[i] = levker_score(&L, prow, pz);
        }
        free(prow); free(pz);
      }
      levker_free(&L);
    }
  }
  if (diag) {
    if (diag->depth_out) *diag->depth_out = depth;
    if (diag->level_sizes)
      for (int l = 0; l <= depth; ++l) diag->level_sizes[l] = lvl_size[l];
    if (diag->level_idx) {
      int64_t off = 0;
      for (int l = 1; l <= depth; ++l) {
        if (off + lvl_size[l] > diag->level_idx_cap) break;
        memcpy(diag->level_idx + off, lvl_ptr[l], sizeof(int64_t) * (size_t)lvl_size[l]);
        off += lvl_size[l];
      }
    }
    if (diag->approx_out) memcpy(diag->approx_out, approx, sizeof(double) * (size_t)(arows * k));
    if (diag->approx_rows) *diag->approx_rows = arows;
    if (diag->scores_out && scores) memcpy(diag->scores_out, scores, sizeof(double) * (size_t)m);
  }
  for (int l = 0; l < nlev; ++l) free(lvl_ptr[l]);
  free(approx);
  double* dist = NULL;
  if (!st) {
    dist = XMALLOC(double, m);
    st = orc_leverage_to_distribution(scores, m, dist);
  }
  if (upfront_seconds) *upfront_seconds = now_seconds() - t0;
  if (!st && !upfront_only) {
    int64_t* idx = XMALLOC(int64_t, c);
    double* wt = XMALLOC(double, c);
    double* a = XMALLOC(double, c * (int64_t)p_bar);
    double* b = XMALLOC(double, c);
    double* phi = XMALLOC(double, p_bar);
    int64_t off = 0;
    for (int p = 1; p <= p_bar && !st; ++p) {
      t0 = now_seconds();
      if (diag && diag->fixed_idx) {
        memcpy(idx, diag->fixed_idx + (int64_t)(p - 1) * c, sizeof(int64_t) * (size_t)c);
        memcpy(wt, diag->fixed_w + (int64_t)(p - 1) * c, sizeof(double) * (size_t)c);
      } else {
        st = orc_sample_rows(dist, m, c, orc_derive_seed(seed, (uint64_t)p), idx, wt);
        if (st) break;
      }
      /* apply_sample(full, s, p): first p columns of the p_bar-wide rows */
      st = orc_apply_sample(y, n, p_bar, idx, wt, c, p, a, b);
      if (!st) st = orc_solve_exact(a, c, p, b, phi, NULL, NULL);
      if (st) break;
      if (lag_seconds) lag_seconds[p - 1] = now_seconds() - t0;
      taus[p - 1] = phi[p - 1];
      if (coefs_packed) memcpy(coefs_packed + off, phi, sizeof(double) * (size_t)p);
      off += p;
      if (diag && diag->idx_out) memcpy(diag->idx_out + (int64_t)(p - 1) * c, idx, sizeof(int64_t) * (size_t)c);
      if (diag && diag->w_out) memcpy(diag->w_out + (int64_t)(p - 1) * c, wt, sizeof(double) * (size_t)c);
    }
    if (!st && p_star) *p_star = orc_select_order(taus, p_bar, 1.96 / sqrt((double)c));
    free(idx); free(wt); free(a); free(b); free(phi);
  }
  free(dist);
  free(scores);
  free(row); free(z); free(sidx); free(sw);
  return st;
}

/* The end of rh_fit replayed from its final approximation (rows arow_idx of
 * the augmented lag-p_bar system, scaled by arow_w, in the order the upward
 * pass gathered them): rh_leverage_scores (repeated_halving.cpp:182-189),
 * leverage_to_distribution and the per-lag draws (:205-220).  With the
 * level-0 upward sample of an orc_rh_fit run the scores and draws are
 * bit-identical to that run. */
int orc_rh_replay(const double* y, int64_t n, int p_bar, int64_t c, uint64_t seed, const int64_t* arow_idx,
                  const double* arow_w, int64_t arows, double* scores_out, int64_t* idx_out, double* w_out) {
  if (p_bar < 1) return fail(ORC_USAGE, "maximum lag must be at least 1");
  if (n <= (int64_t)p_bar + 1) return fail(ORC_DATA, "series too short for maximum lag %d", p_bar);
  const int64_t m = n - p_bar, k = p_bar + 1;
  double* approx = XMALLOC(double, arows * k);
  double* row = XMALLOC(double, k);
  for (int64_t t = 0; t < arows; ++t) {
    aug_row(y, p_bar, arow_idx[t], row);
    for (int64_t j = 0; j < k; ++j) approx[j * arows + t] = arow_w ? row[j] * arow_w[t] : row[j];
  }
  levker_t L;
  int st = levker_init(&L, approx, arows, k, 0, 0);
  double* scores = XMALLOC(double, m);
  if (!st) {
#pragma omp parallel
    {
      double* prow = XMALLOC(double, k);
      double* pz = XMALLOC(double, k);
#pragma omp for schedule(static)
      for (int64_t i = 0; i < m; ++i) {
        aug_row(y, p_bar, i, prow);
        scores[i] = levker_score(&L, prow, pz);
      }
      free(prow); free(pz);
    }
    levker_free(&L);
  }
  double* dist = XMALLOC(double, m);
  if (!st && scores_out) memcpy(scores_out, scores, sizeof(double) * (size_t)m);
  if (!st) st = orc_leverage_to_distribution(scores, m, dist);
  for (int p = 1; p <= p_bar && !st; ++p)
    st = orc_sample_rows(dist, m, c, orc_derive_seed(seed, (uint64_t)p), idx_out + (int64_t)(p - 1) * c,
                         w_out + (int64_t)(p - 1) * c);
  free(approx); free(row); free(scores); free(dist);
  return st;
}

int orc_rh_fit(const double* y, int64_t n, int p_bar, int64_t c, const orc_rh_cfg* cfg_in,
               uint64_t seed, orc_rh_diag* diag, double* taus, double* coefs_packed,
               double* lag_seconds, double* upfront_seconds, int* p_star) {
  return rh_fit_impl(y, n, p_bar, c, cfg_in, seed, diag, taus, coefs_packed, lag_seconds,
                     upfront_seconds, p_star, 0);
}

/* bench timing helper: the RH upfront phase alone (halving, upward sampling,
 * final scores and distribution), default configuration. */
double orc_rh_time_upfront(const double* y, int64_t n, int p_bar, int64_t c, uint64_t seed) {
  double up = -1.0;
  if (rh_fit_impl(y, n, p_bar, c, NULL, seed, NULL, NULL, NULL, NULL, &up, NULL, 1)) return -1.0;
  return up;
}

/* ======================================================================
 * bench.cpp:27-48 exact per-lag OLS on the full series
 * ==================================================================== */
int orc_exact_fit(const double* y, int64_t n, int p_bar, double* taus, double* coefs_packed,
                  int* p_star) {
  if (p_bar < 1) return fail(ORC_USAGE, "maximum lag must be at least 1");
  if (n <= (int64_t)p_bar + 1) return fail(ORC_DATA, "series too short for maximum lag %d", p_bar);
  int64_t off = 0;
  for (int h = 1; h <= p_bar; ++h) {
    const int64_t m = n - h;
    double* a = XMALLOC(double, m * h);
    double* phi = XMALLOC(double, h);
    for (int j = 0; j < h; ++j)
      for (int64_t i = 0; i < m; ++i) a[(int64_t)j * m + i] = y[h - 1 - j + i];
    orc_solve_exact(a, m, h, y + h, phi, NULL, NULL);
    taus[h - 1] = phi[h - 1];
    if (coefs_packed) memcpy(coefs_packed + off, phi, sizeof(double) * (size_t)h);
    off += h;
    free(a);
    free(phi);
  }
  if (p_star) *p_star = orc_select_order(taus, p_bar, 1.96 / sqrt((double)n - p_bar));
  return ORC_OK;
}

/* ======================================================================
 * SRHT path: sketch.cpp:103-239, bench.cpp:50-72
 * ==================================================================== */
#define INV_SQRT2 0.70710678118654752440

/* sketch.cpp:107-120: in place, strides 1, 2, 4, ... (n a power of two) */
int orc_hadamard_apply(double* x, int64_t n) {
  if (n == 0 || (n & (n - 1)) != 0) return fail(ORC_USAGE, "transform length must be a power of two");
  for (int64_t h = 1; h < n; h <<= 1)
    for (int64_t i = 0; i < n; i += 2 * h)
      for (int64_t j = i; j < i + h; ++j) {
        const double a = x[j], b = x[j + h];
        x[j] = (a + b) * INV_SQRT2;
        x[j + h] = (a - b) * INV_SQRT2;
      }
  return ORC_OK;
}

/* sketch.cpp:145-163 (PartialHadamard::recurse): largest stride first, only
 * the halves that hold requested rows; idx sorted unique, relative to x */
static void partial_recurse(const double* x, int64_t len, const int64_t* idx, int64_t nidx, double* out,
                            const int64_t* outpos, double* scratch) {
  if (nidx == 0) return;
  if (len == 1) {
    for (int64_t r = 0; r < nidx; ++r) out[outpos[r]] = x[0];
    return;
  }
  const int64_t h = len / 2;
  int64_t mid = 0;
  while (mid < nidx && idx[mid] < h) ++mid;
  double* buf = scratch;  /* this level's buffer (len / 2), deeper levels after it */
  if (mid > 0) {
    for (int64_t i = 0; i < h; ++i) buf[i] = (x[i] + x[i + h]) * INV_SQRT2;
    partial_recurse(buf, h, idx, mid, out, outpos, scratch + h);
  }
  if (mid < nidx) {
    for (int64_t i = 0; i < h; ++i) buf[i] = (x[i] - x[i + h]) * INV_SQRT2;
    int64_t* shifted = XMALLOC(int64_t, nidx - mid);
    for (int64_t r = mid; r < nidx; ++r) shifted[r - mid] = idx[r] - h;
    partial_recurse(buf, h, shifted, nidx - mid, out, outpos + mid, scratch + h);
    free(shifted);
  }
}

/* sketch.cpp:165-185 */
int orc_srht_sample_count(int64_t n, int64_t d, double epsilon, double* formula_value, int64_t* c,
                          int* capped) {
  if (!(n > d && d >= 1)) return fail(ORC_USAGE, "need n > d >= 1");
  if (!(epsilon > 0.0 && epsilon < 1.0)) return fail(ORC_USAGE, "epsilon must lie in (0, 1)");
  const double nd = (double)n * (double)d;
  const double log_term = log(40.0 * nd);
  const double branch1 = 48.0 * 48.0 * (double)d * log_term * log(100.0 * 100.0 * d * log_term);
  const double branch2 = 40.0 * (double)d * log_term / epsilon;
  *formula_value = branch1 > branch2 ? branch1 : branch2;
  const double rounded = ceil(*formula_value);
  if (rounded > (double)n) {
    *c = n;
    *capped = 1;
  } else {
    *c = (int64_t)rounded;
    *capped = 0;
  }
  return ORC_OK;
}

static uint64_t bit_ceil_u64(uint64_t v) {
  uint64_t n = 1;
  while (n < v) n <<= 1;
  return n;
}

/* sketch.cpp:187-239.  a: rows x cols, column-major.  sa / sb (optional)
 * receive the sampled, weighted c x cols system (column-major) */
int orc_srht_solve(const double* a, int64_t n0, int64_t d, const double* b, int64_t c, uint64_t seed,
                   double* x, double* sa, double* sb) {
  if (n0 < d) return fail(ORC_USAGE, "need rows >= columns");
  if (c < d) return fail(ORC_USAGE, "sample count below column count");
  const int64_t n = (int64_t)bit_ceil_u64((uint64_t)n0);
  orc_rng rng;
  orc_rng_init(&rng, seed);
  double* sign = XMALLOC(double, n0);
  for (int64_t i = 0; i < n0; ++i) sign[i] = (orc_rng_next(&rng) >> 63) ? 1.0 : -1.0;
  int64_t* draws = XMALLOC(int64_t, c);
  for (int64_t t = 0; t < c; ++t) draws[t] = (int64_t)orc_rng_below(&rng, (uint64_t)n);
  int64_t* uniq = XMALLOC(int64_t, c);
  for (int64_t t = 0; t < c; ++t) uniq[t] = draws[t];
  qsort(uniq, (size_t)c, sizeof(int64_t), cmp_i64);
  int64_t nu = 0;
  for (int64_t t = 0; t < c; ++t)
    if (nu == 0 || uniq[t] != uniq[nu - 1]) uniq[nu++] = uniq[t];
  int64_t* outpos = XMALLOC(int64_t, nu);
  for (int64_t k = 0; k < nu; ++k) outpos[k] = k;
  double* padded = XMALLOC(double, n);
  double* scratch = XMALLOC(double, n);
  double* vals = XMALLOC(double, nu);
  int64_t* posof = XMALLOC(int64_t, c);
  for (int64_t t = 0; t < c; ++t) { /* lower_bound in uniq */
    int64_t lo = 0, hi = nu;
    while (lo < hi) {
      const int64_t m = (lo + hi) / 2;
      if (uniq[m] < draws[t]) lo = m + 1;
      else hi = m;
    }
    posof[t] = lo;
  }
  const double w = sqrt((double)n / (double)c);
  double* as = sa ? sa : XMALLOC(double, c * d);
  double* bs = sb ? sb : XMALLOC(double, c);
  for (int64_t j = 0; j <= d; ++j) {
    const double* col = j < d ? a + j * n0 : b;
    for (int64_t i = 0; i < n0; ++i) padded[i] = sign[i] * col[i];
    for (int64_t i = n0; i < n; ++i) padded[i] = 0.0;
    partial_recurse(padded, n, uniq, nu, vals, outpos, scratch);
    double* dst = j < d ? as + j * c : bs;
    for (int64_t t = 0; t < c; ++t) dst[t] = w * vals[posof[t]];
  }
  const int rc = orc_solve_exact(as, c, d, bs, x, NULL, NULL);
  if (!sa) free(as);
  if (!sb) free(bs);
  free(sign); free(draws); free(uniq); free(outpos); free(padded); free(scratch); free(vals); free(posof);
  return rc;
}

/* bench.cpp:50-72 */
int orc_srht_fit(const double* y, int64_t n, int p_bar, int64_t c, uint64_t seed, double* taus,
                 double* coefs_packed, int* p_star) {
  if (p_bar < 1) return fail(ORC_USAGE, "maximum lag must be at least 1");
  if (n <= (int64_t)p_bar + 1) return fail(ORC_DATA, "series too short for maximum lag %d", p_bar);
  if (c < p_bar) return fail(ORC_USAGE, "sample count below maximum lag");
  int64_t off = 0;
  for (int h = 1; h <= p_bar; ++h) {
    const int64_t m = n - h;
    double* a = XMALLOC(double, m * h);
    double* phi = XMALLOC(double, h);
    for (int j = 0; j < h; ++j)
      for (int64_t i = 0; i < m; ++i) a[(int64_t)j * m + i] = y[h - 1 - j + i];
    const int rc = orc_srht_solve(a, m, h, y + h, c, orc_derive_seed(seed, (uint64_t)h), phi, NULL, NULL);
    if (rc != ORC_OK) {
      free(a);
      free(phi);
      return rc;
    }
    taus[h - 1] = phi[h - 1];
    if (coefs_packed) memcpy(coefs_packed + off, phi, sizeof(double) * (size_t)h);
    off += h;
    free(a);
    free(phi);
  }
  if (p_star) *p_star = orc_select_order(taus, p_bar, 1.96 / sqrt((double)c));
  return ORC_OK;
}

/* ======================================================================
 * series.cpp:58-107 -- reference generators (test inputs only)
 * ==================================================================== */
int orc_partials_to_ar(const double* partials, int p, double* phi) {
  double* cur = XMALLOC(double, p);
  double* nxt = XMALLOC(double, p);
  for (int k = 0; k < p; ++k) {
    const double kappa = partials[k];
    if (!(fabs(kappa) < 1.0)) {
      free(cur); free(nxt);
      return fail(ORC_USAGE, "partial autocorrelation at lag %d is outside (-1, 1)", k + 1);
    }
    for (int j = 0; j < k; ++j) nxt[j] = cur[j] - kappa * cur[k - 1 - j];
    nxt[k] = kappa;
    double* t = cur; cur = nxt; nxt = t;
  }
  memcpy(phi, cur, sizeof(double) * (size_t)p);
  free(cur); free(nxt);
  return ORC_OK;
}

int orc_random_stationary_ar(int p, uint64_t seed, double* phi) {
  if (p < 1) return fail(ORC_USAGE, "model order must be at least 1");
  orc_rng rng;
  orc_rng_init(&rng, seed);
  double* partials = XMALLOC(double, p);
  for (int k = 0; k < p; ++k) partials[k] = rng_uniform(&rng, -0.9, 0.9);
  while (fabs(partials[p - 1]) < 0.1) partials[p - 1] = rng_uniform(&rng, -0.9, 0.9);
  int st = orc_partials_to_ar(partials, p, phi);
  free(partials);
  return st;
}

int orc_simulate_ar(const double* phi, int p, double noise_std, int64_t n, int64_t burn_in,
                    uint64_t seed, double* out) {
  if (n == 0) return fail(ORC_USAGE, "cannot simulate an empty series");
  orc_rng rng;
  orc_rng_init(&rng, seed);
  double* state = XMALLOC(double, p);
  for (int j = 0; j < p; ++j) state[j] = 0.0;
  for (int64_t t = 0; t < burn_in + n; ++t) {
    double v = noise_std == 0.0 ? 0.0 : noise_std * orc_rng_normal(&rng);
    for (int j = 0; j < p; ++j) v += phi[j] * state[j];
    for (int j = p - 1; j > 0; --j) state[j] = state[j - 1];
    if (p > 0) state[0] = v;
    if (t >= burn_in) out[t - burn_in] = v;
  }
  free(state);
  return ORC_OK;
}
