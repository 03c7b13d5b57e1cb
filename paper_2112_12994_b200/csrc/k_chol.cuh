// k_chol.cuh -- small dense factorizations of the CholeskyQR solve.
//
// The reference solves each sampled system with Eigen's ColPivHouseholderQR
// (toeplitz.cpp:57-71).  Here the c x (p+1) augmented system [A b] is
// factored by (shifted) CholeskyQR2/3 -- GEMM-shaped, tensor-core friendly --
// and the p x p back-substitutions operate on K = p+1 sized factors:
//   k_chol   : single CTA, blocked (32) right-looking Cholesky G = R^T R of
//              one Gram matrix, A held packed in shared memory.  On a
//              non-positive pivot in iteration 1 it restarts with the
//              Fukaya et al. shift 11 (cK + K(K+1)) eps tr(G) and flags the
//              lag for a third CholeskyQR iteration.
//   k_trinv  : R^-1 columns, one warp per column (row-oriented substitution),
//              written dense (rows optionally permuted to the gathered
//              column order the Q-formation kernel consumes).
//   k_phi    : phi = R_A^-1 z from the chain R = R_n ... R_1:
//                v_n = -Rinv_n[:p,p] / Rinv_n[p,p]
//                v_i = (Rinv_i[:p,:p] v_{i+1} - Rinv_i[:p,p]) / Rinv_i[p,p]
//              phi = v_1; tau_p = phi[p-1] (lsar.cpp:117).
#pragma once

#include "common.cuh"
#include "k_sample.cuh"

namespace tfk {

constexpr int kCholThreads = 1024;
constexpr int kCholSmemLimit = 227 * 1024 - 1024;  // leave room for static smem

__device__ __forceinline__ int pcol(int i, int j) { return ((j * (j + 1)) >> 1) + i; }
__host__ __device__ __forceinline__ int64_t prow_off(int r, int K) {
  return (int64_t)r * K - ((int64_t)r * (r - 1)) / 2;
}
__host__ __device__ __forceinline__ int gperm(int a, int K) { return a < K - 1 ? a + 1 : 0; }

inline size_t chol_smem_bytes(int K) {
  return sizeof(double) * ((size_t)K * (K + 1) / 2 + 32 * 33 + 8);
}
inline bool chol_fits_smem(int K) { return chol_smem_bytes(K) <= (size_t)kCholSmemLimit; }

struct CholArgs {
  const double* G;   // dense row-major K x K (upper valid)
  int K;
  int perm;          // 1: G is in gathered column order (target first)
  int iter;          // 1, 2, 3 (3 runs only when flags[0] != 0)
  int64_t nrows;     // rows of the tall matrix (shift formula)
  int use_smem;
  double* ws;        // global packed scratch when !use_smem
  double* Rrow;      // out: packed row-major upper R
  int* flags;        // [0] shifted (written by iter 1), [1] failed
  int* status;
  int lag;
};

__global__ void __launch_bounds__(kCholThreads) k_chol(CholArgs a) {
  extern __shared__ double smem[];
  __shared__ int s_bad;
  const int K = a.K;
  if (a.iter == 3 && a.flags[0] == 0) return;
  if (a.iter > 1 && a.flags[1] != 0) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int tri = K * (K + 1) / 2;
  double* A = a.use_smem ? smem : a.ws;
  double* Dv = a.use_smem ? smem + tri : smem;
  double shift = 0.0;
  int shifted = 0;
  double trace = 0.0;
  for (int i = 0; i < K; ++i) {
    const int gi = a.perm ? gperm(i, K) : i;
    trace += a.G[(size_t)gi * K + gi];
  }
  const double pivot_floor = 4.930380657631324e-32 * trace;
  for (int attempt = 0; attempt < 2; ++attempt) {
    for (int j = warp; j < K; j += 32)
      for (int i = lane; i <= j; i += 32) {
        const int gi = a.perm ? gperm(i, K) : i, gj = a.perm ? gperm(j, K) : j;
        const int lo = min(gi, gj), hi = max(gi, gj);
        double g = a.G[(size_t)lo * K + hi];
        if (i == j) g += shift;
        A[pcol(i, j)] = g;
      }
    if (tid == 0) s_bad = 0;
    __syncthreads();
    for (int b0 = 0; b0 < K; b0 += 32) {
      const int m = min(32, K - b0);
      if (warp == 0) {
        for (int i = 0; i < m; ++i) {
          double d = 0.0;
          if (lane == i) {
            double g = A[pcol(b0 + i, b0 + i)];
            if (b0 + i == K - 1 && !(g > pivot_floor)) g = pivot_floor;  // see k_cholinv.cuh
            if (!(g > 0.0) || !isfinite(g)) s_bad = 1;
            d = sqrt(fmax(g, 0.0));
            A[pcol(b0 + i, b0 + i)] = d;
          }
          d = __shfl_sync(0xffffffffu, d, i);
          if (lane > i && lane < m) A[pcol(b0 + i, b0 + lane)] /= d;
          __syncwarp();
          if (lane > i && lane < m) {
            const double rij = A[pcol(b0 + i, b0 + lane)];
            for (int r = i + 1; r <= lane; ++r) A[pcol(b0 + r, b0 + lane)] -= A[pcol(b0 + i, b0 + r)] * rij;
          }
          __syncwarp();
        }
        if (lane < m) {  // Dinv(r, l) = (R_bb^-1)(r, l), column l per lane
          const int l = lane;
          Dv[l * 33 + l] = 1.0 / A[pcol(b0 + l, b0 + l)];
          for (int r = l - 1; r >= 0; --r) {
            double s = 0.0;
            for (int q = r + 1; q <= l; ++q) s += A[pcol(b0 + r, b0 + q)] * Dv[q * 33 + l];
            Dv[r * 33 + l] = -s / A[pcol(b0 + r, b0 + r)];
          }
        }
      }
      __syncthreads();
      if (s_bad) break;
      // panel row: R(b, j) = R_bb^-T G(b, j) for j beyond the block
      const int nc = K - b0 - m;
      const int total = m * nc;
      for (int base = 0; base < total; base += kCholThreads * 8) {
        double vals[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int e = base + u * kCholThreads + tid;
          vals[u] = 0.0;
          if (e < total) {
            const int r = e % m, j = b0 + m + e / m;
            double s = 0.0;
            for (int q = 0; q <= r; ++q) s += Dv[q * 33 + r] * A[pcol(b0 + q, j)];
            vals[u] = s;
          }
        }
        __syncthreads();
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int e = base + u * kCholThreads + tid;
          if (e < total) A[pcol(b0 + e % m, b0 + m + e / m)] = vals[u];
        }
        __syncthreads();
      }
      // trailing update of the Schur complement
      for (int j = b0 + m + warp; j < K; j += 32) {
        const int cj = pcol(b0, j);
        for (int i = b0 + m + lane; i <= j; i += 32) {
          const int ci = pcol(b0, i);
          double s = 0.0;
          for (int r = 0; r < m; ++r) s = fma(A[ci + r], A[cj + r], s);
          A[pcol(i, j)] -= s;
        }
      }
      __syncthreads();
    }
    if (!s_bad) break;
    if (a.iter == 1 && !shifted) {
      // shifted CholeskyQR restart (Fukaya, Kannan, Nakatsukasa, Yamamoto, Yanagisawa 2020)
      shift = 11.0 * ((double)a.nrows * K + (double)K * (K + 1)) * 2.220446049250313e-16 * trace;
      shifted = 1;
      __syncthreads();
      continue;
    }
    if (tid == 0) {
      a.flags[1] = 1;
      raise_status(a.status, kErrNumerical, a.lag, kReasonCholFail);
    }
    return;
  }
  if (a.iter == 1 && tid == 0) {
    a.flags[0] = shifted;
    a.flags[1] = 0;
  }
  for (int j = warp; j < K; j += 32)
    for (int i = lane; i <= j; i += 32) a.Rrow[prow_off(i, K) + (j - i)] = A[pcol(i, j)];
}

// ---------------------------------------------------------------------------
constexpr int kTrinvWarps = 16;

// X = R^-1 (upper) for columns [0, K); column l computed by one warp:
//   x_l = 1/R(l,l);  x_r = -(sum_{q=r+1..l} R(r,q) x_q) / R(r,r)
// out[(perm ? gperm(q) : q) * K + l] = x_q  (x_q = 0 for q > l)
template <int SLOTS>
__global__ void __launch_bounds__(kTrinvWarps * 32)
    k_trinv(const double* __restrict__ Rrow, int K, int perm, double* __restrict__ out,
            const int* gate) {
  if (gate && *gate == 0) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int l = blockIdx.x * kTrinvWarps + warp;
  if (l >= K) return;
  double xs[SLOTS];
#pragma unroll
  for (int s = 0; s < SLOTS; ++s) xs[s] = 0.0;
  for (int r = l; r >= 0; --r) {
    const double* Rr = Rrow + prow_off(r, K) - r;  // Rr[q] = R(r, q), q >= r
    double part = 0.0;
#pragma unroll
    for (int s = 0; s < SLOTS; ++s) {
      const int q = lane + 32 * s;
      if (q > r && q <= l) part = fma(Rr[q], xs[s], part);
    }
    const double sum = warp_sum(part);
    const double xr = ((r == l ? 1.0 : 0.0) - sum) / Rr[r];
#pragma unroll
    for (int s = 0; s < SLOTS; ++s)
      if (lane + 32 * s == r) xs[s] = xr;
  }
#pragma unroll
  for (int s = 0; s < SLOTS; ++s) {
    const int q = lane + 32 * s;
    if (q < K) out[(size_t)(perm ? gperm(q, K) : q) * K + l] = q <= l ? xs[s] : 0.0;
  }
}

// ---------------------------------------------------------------------------
struct PhiArgs {
  int K;                 // p + 1
  const double* Rg1;     // dense Rinv_1, rows in gathered order
  const double* Rinv2;   // dense Rinv_2 (aug order)
  const double* Rinv3;   // dense Rinv_3 (aug order), valid when shifted
  const int* flags;
  double* phi;           // out: length p
  double* coefs;         // packed coefficient array (nullable)
  int64_t coef_off;
  double* taus;          // nullable
  int* method;           // nullable, per lag
  int lag;               // 1-based index of this lag in the output arrays
};

constexpr int kPhiThreads = 1024;

// phi = R_A^-1 z for R = R_n ... R_1 (see file header)
__global__ void __launch_bounds__(kPhiThreads) k_phi(PhiArgs a) {
  extern __shared__ double sm[];  // v[K], u[K]
  const int K = a.K, p = K - 1;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double* v = sm;
  double* u = sm + K;
  if (a.flags[1]) {
    for (int q = tid; q < p; q += kPhiThreads) a.phi[q] = __longlong_as_double(0x7ff8000000000000ll);
    return;
  }
  const int shifted = a.flags[0];
  const double* Rn = shifted ? a.Rinv3 : a.Rinv2;
  const double xp = Rn[(size_t)p * K + p];
  for (int q = tid; q < p; q += kPhiThreads) v[q] = -Rn[(size_t)q * K + p] / xp;
  __syncthreads();
  for (int it = shifted ? 2 : 1; it >= 1; --it) {
    for (int q = warp; q < p; q += kPhiThreads / 32) {
      const double* row = it == 1 ? a.Rg1 + (size_t)gperm(q, K) * K : a.Rinv2 + (size_t)q * K;
      double part = 0.0;
      for (int l = q + lane; l < p; l += 32) part = fma(row[l], v[l], part);
      const double s = warp_sum(part);
      if (lane == 0) u[q] = s - row[p];
    }
    __syncthreads();
    const double dpp = it == 1 ? a.Rg1[(size_t)gperm(p, K) * K + p] : a.Rinv2[(size_t)p * K + p];
    for (int q = tid; q < p; q += kPhiThreads) v[q] = u[q] / dpp;
    __syncthreads();
  }
  for (int q = tid; q < p; q += kPhiThreads) {
    a.phi[q] = v[q];
    if (a.coefs) a.coefs[a.coef_off + q] = v[q];
  }
  if (tid == 0) {
    if (a.taus) a.taus[a.lag - 1] = v[p - 1];
    if (a.method) a.method[a.lag - 1] = shifted ? 2 : 0;
  }
}

// p = 1: a single lag column is perfectly conditioned, so the normal equation
// phi = a^T b / a^T a is as accurate as Householder -- and, like the
// reference's Householder solve, exact when b is an exact power-of-two
// multiple of a (the zero-residual case of test_lsar.cpp:160-169).
__global__ void k_solve_k2(const double* G, PhiArgs a) {
  // gathered order: column 0 = target b, column 1 = lag column a
  const double phi = G[1] / G[3];
  a.phi[0] = phi;
  if (a.coefs) a.coefs[a.coef_off] = phi;
  if (a.taus) a.taus[a.lag - 1] = phi;
  if (a.method) a.method[a.lag - 1] = 0;
}

}  // namespace tfk
