// k_cholinv.cuh -- fused Cholesky factorization + triangular inverse of one
// K x K Gram matrix in a single CTA, K <= kCholinvMaxK (all of C1-C3).
//
// G = R^T R (upper R), output Rinv = R^-1 (dense, row-major, lower part 0,
// rows optionally permuted to the gathered column order).  This is the small
// dense core of each CholeskyQR iteration that replaces Eigen's
// ColPivHouseholderQR (toeplitz.cpp:57-71) on the sampled system.
//
// Storage: the upper triangle as 32 x 32 tiles ("tile-packed"), each tile
// column-major with leading dimension 36 (conflict-free DMMA fragment loads),
// last tile column only as wide as needed -> 207 KB of shared memory at K=201.
//
// Blocked right-looking Cholesky, block 32:
//   1. warp 0 factors the diagonal tile in registers (lane l owns column l,
//      row broadcasts by shuffles) and inverts it in registers; the diagonal
//      tile is overwritten by Dinv_b = R_bb^-1.
//   2. panel:    R(b, J)  = Dinv_b^T G(b, J)            (DMMA m8n8k4 f64)
//   3. trailing: G(I, J) -= R(b, I)^T R(b, J)           (DMMA)
// In-place blocked inverse, row blocks bottom-up:
//   W(I, L)    = -Dinv_I R(I, L)                        (DMMA)
//   Rinv(I, J) = sum_{L=I+1..J} W(I, L) Rinv(L, J)       (DMMA)
// A non-positive pivot in CholeskyQR iteration 1 restarts the factorization
// with the shift 11 (cK + K(K+1)) eps tr(G) (shifted CholeskyQR3).
#pragma once

#ifndef CI_STAMP
#define CI_STAMP(k) ((void)0)
#endif

#include "common.cuh"
#include "k_chol.cuh"
#include "k_sample.cuh"

namespace tfk {

constexpr int kCI_T = 32;
constexpr int kCI_LD = 36;
constexpr int kCholinvMaxK = 211;  // (21*32 + 7*19) tile columns * 36 * 8 B <= 227 KB
constexpr int kCholinvMaxNB = (kCholinvMaxK + 31) / 32;
constexpr int kCholinvThreads = 256;  // 8 warps: 255 registers for the register-resident diagonal block
constexpr int kCI_W = kCholinvThreads / 32;

__host__ __device__ inline int ci_tw(int J, int K) { return min(32, K - 32 * J); }

__host__ inline size_t cholinv_smem_bytes(int K) {
  const int nb = (K + 31) / 32;
  size_t tot = 0;
  for (int J = 0; J < nb; ++J) tot += (size_t)(J + 1) * ci_tw(J, K) * kCI_LD;
  return tot * sizeof(double);
}

struct CholinvArgs {
  const double* G;   // dense row-major K x K (upper valid)
  int K;
  int perm_in;       // G in gathered column order (target first)
  int perm_out;      // write Rinv rows in gathered order
  int iter;          // 1, 2, 3 (3 runs only when flags[0] != 0)
  int64_t nrows;     // rows of the tall matrix (shift formula)
  double* Rinv;      // out: dense row-major K x K
  int* flags;        // [0] shifted (written by iter 1), [1] failed
  int* status;
  int lag;
};

struct CITiles {
  double* base;
  int K, nb;
  const int* off;  // shared-memory table of tile-column offsets
  __device__ __forceinline__ double* tile(int I, int J) const {
    return base + off[J] + I * ci_tw(J, K) * kCI_LD;
  }
};

// acc (32 x 16 output: rows 0..31, cols n0..n0+15) += sum_k A(m, k) B(k, n), k in [0, 32)
template <class FA, class FB>
__device__ __forceinline__ void ci_mma(double (&acc)[4][2][2], int n0, FA fa, FB fb) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int kk = 0; kk < 8; ++kk) {
    const int k = 4 * kk + (lane & 3);
    double a[4], b[2];
#pragma unroll
    for (int i = 0; i < 4; ++i) a[i] = fa(8 * i + (lane >> 2), k);
#pragma unroll
    for (int j = 0; j < 2; ++j) b[j] = fb(k, n0 + 8 * j + (lane >> 2));
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], a[i], b[j]);
  }
}

__device__ __forceinline__ void ci_zero(double (&acc)[4][2][2]) {
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
}

// store (or subtract) a 32 x 16 accumulator into a tile with width w
template <int MODE>  // 0 store, 1 subtract, 2 store negated
__device__ __forceinline__ void ci_put(double* t, int w, int n0, const double (&acc)[4][2][2]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int r = 8 * i + (lane >> 2), c = n0 + 8 * j + 2 * (lane & 3) + e;
        if (c < w) {
          double* p = t + c * kCI_LD + r;
          if (MODE == 0) *p = acc[i][j][e];
          else if (MODE == 1) *p -= acc[i][j][e];
          else *p = -acc[i][j][e];
        }
      }
}

// Factor + invert the diagonal tile (b, b) in shared memory with one warp
// (lane l owns column l); compact loop code -- a fully unrolled register
// version was ~40k instructions and its instruction-cache misses dominated.
// Row i is published to a separate buffer each step so the compiler can
// batch the loads of an update (no aliasing with the column being written).
// The tile is overwritten by Dinv_b = R_bb^-1; returns true on a bad pivot.
// `last` = local index of the augmented target column (or -1): a vanishing
// residual (c == p) gives a non-positive last pivot, clamped to `floor` --
// phi depends only on Rinv[:p,p] / Rinv[p,p], which any positive pivot keeps.
__device__ __noinline__ bool ci_diag(double* __restrict__ D, double* __restrict__ rowbuf, int m,
                                     int last, double floor) {
  const int lane = threadIdx.x & 31;
  bool bad = false;
  double* __restrict__ col = D + lane * kCI_LD;  // column `lane`
  const bool mine = lane < m;
  CI_STAMP(50);
  for (int i = 0; i < m; ++i) {
    double piv = D[i * kCI_LD + i];
    if (i == last && !(piv > floor)) piv = floor;
    bad |= !(piv > 0.0) || !isfinite(piv);
    const double inv = fast_rsqrt(piv);
    __syncwarp();
    double ril = 0.0;
    if (lane == i) col[i] = piv * inv;
    else if (lane > i && mine) {
      ril = col[i] * inv;
      col[i] = ril;
      rowbuf[lane] = ril;
    }
    __syncwarp();
    if (lane > i && mine) {
      int r = i + 1;
      for (; r + 3 <= lane; r += 4) {
        const double a0 = rowbuf[r], a1 = rowbuf[r + 1], a2 = rowbuf[r + 2], a3 = rowbuf[r + 3];
        const double c0 = col[r], c1 = col[r + 1], c2 = col[r + 2], c3 = col[r + 3];
        col[r] = fma(-a0, ril, c0);
        col[r + 1] = fma(-a1, ril, c1);
        col[r + 2] = fma(-a2, ril, c2);
        col[r + 3] = fma(-a3, ril, c3);
      }
      for (; r <= lane; ++r) col[r] = fma(-rowbuf[r], ril, col[r]);
    }
  }
  __syncwarp();
  CI_STAMP(51);
  // in-place inverse, rows bottom-up: x(i,l) = (delta_il - sum_{q>i} R(i,q) x(q,l)) / R(i,i)
  // (row i of R is dead once row i of X is written; column l stays in lane l)
  for (int i = m - 1; i >= 0; --i) {
    if (lane > i && mine) rowbuf[lane] = col[i];  // R(i, lane)
    __syncwarp();
    double a0 = (lane == i) ? 1.0 : 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    if (lane >= i && mine) {
      int q = i + 1;
      for (; q + 3 <= lane; q += 4) {
        a0 = fma(-rowbuf[q], col[q], a0);
        a1 = fma(-rowbuf[q + 1], col[q + 1], a1);
        a2 = fma(-rowbuf[q + 2], col[q + 2], a2);
        a3 = fma(-rowbuf[q + 3], col[q + 3], a3);
      }
      for (; q <= lane; ++q) a0 = fma(-rowbuf[q], col[q], a0);
    }
    const double rinv = fast_rcp(D[i * kCI_LD + i]);
    __syncwarp();
    if (lane >= i && mine) col[i] = ((a0 + a1) + (a2 + a3)) * rinv;
    __syncwarp();
  }
  CI_STAMP(52);
  if (mine)
    for (int r = lane + 1; r < 32; ++r) col[r] = 0.0;  // strictly lower part
  return __any_sync(0xffffffffu, bad);
}

// SYRK update of one half tile: C(I, J)[:, n0:n0+16] -= R(b, I)^T R(b, J)
__device__ __forceinline__ void ci_syrk_item(const CITiles& T, int b, int I, int J, int n0) {
  const int K = T.K;
  const int wI = ci_tw(I, K), wJ = ci_tw(J, K);
  const double* pI = T.tile(b, I);
  const double* pJ = T.tile(b, J);
  double acc[4][2][2];
  ci_zero(acc);
  ci_mma(acc, n0, [&](int mm, int k) { return mm < wI ? pI[mm * kCI_LD + k] : 0.0; },
         [&](int k, int n) { return n < wJ ? pJ[n * kCI_LD + k] : 0.0; });
  ci_put<1>(T.tile(I, J), wJ, n0, acc);
}

__global__ void __launch_bounds__(kCholinvThreads) k_cholinv(CholinvArgs a) {
  extern __shared__ __align__(16) double smem[];
  __shared__ int s_bad;
  __shared__ int s_off[kCholinvMaxNB + 1];
  __shared__ double s_tr;
  __shared__ double s_rowbuf[32];
  const int K = a.K;
  if (a.iter == 3 && a.flags[0] == 0) return;
  if (a.iter > 1 && a.flags[1] != 0) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  CI_STAMP(0);
  CITiles T;
  T.base = smem;
  T.K = K;
  T.nb = (K + 31) / 32;
  T.off = s_off;
  const int nb = T.nb;
  if (tid == 0) {
    int acc = 0;
    for (int J = 0; J < nb; ++J) {
      s_off[J] = acc;
      acc += (J + 1) * ci_tw(J, K) * kCI_LD;
    }
    s_off[nb] = acc;
  }
  if (warp == 1) {  // trace of G (augmented order), fixed-order warp reduction
    double t = 0.0;
    for (int i = lane; i < K; i += 32) {
      const int gi = a.perm_in ? gperm(i, K) : i;
      t += a.G[(size_t)gi * K + gi];
    }
    t = warp_sum(t);
    if (lane == 0) s_tr = t;
  }
  __syncthreads();
  const double tr = s_tr;
  const double pivot_floor = 4.930380657631324e-32 * tr;  // (eps)^2 tr(G)
  double shift = 0.0;
  int shifted = 0;

  for (int attempt = 0; attempt < 2; ++attempt) {
    // ---- load the upper triangle into the tiles (rows by warps, no division) ----
    for (int e = tid; e < s_off[nb]; e += kCholinvThreads) smem[e] = 0.0;
    __syncthreads();
    for (int gi = warp; gi < K; gi += kCI_W) {
      const int pi = a.perm_in ? gperm(gi, K) : gi;
      const int I = gi >> 5, ri = gi & 31;
      for (int gj = gi + lane; gj < K; gj += 32) {
        const int pj = a.perm_in ? gperm(gj, K) : gj;
        double v = __ldg(a.G + (size_t)min(pi, pj) * K + max(pi, pj));
        if (gi == gj) v += shift;
        const int J = gj >> 5;
        T.tile(I, J)[(gj & 31) * kCI_LD + ri] = v;
      }
    }
    if (tid == 0) s_bad = 0;
    __syncthreads();
    CI_STAMP(1);
    if (warp == 0 && ci_diag(T.tile(0, 0), s_rowbuf, ci_tw(0, K), nb == 1 ? ci_tw(0, K) - 1 : -1, pivot_floor) && lane == 0) s_bad = 1;
    __syncthreads();

    for (int b = 0; b < nb && !s_bad; ++b) {
      const double* Db = T.tile(b, b);
      // ---- panel: R(b, J) = Dinv_b^T G(b, J), J > b (two-phase, in place) ----
      {
        const int nitems = (nb - 1 - b) * 2;
        double acc[2][4][2][2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int it = warp + h * kCI_W;
          const int J = b + 1 + (it >> 1), n0 = 16 * (it & 1);
          if (it < nitems && n0 < ci_tw(J, K)) {
            const int wJ = ci_tw(J, K);
            const double* tj = T.tile(b, J);
            ci_zero(acc[h]);
            ci_mma(acc[h], n0, [&](int mm, int k) { return Db[mm * kCI_LD + k]; },
                   [&](int k, int n) { return n < wJ ? tj[n * kCI_LD + k] : 0.0; });
          }
        }
        __syncthreads();
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int it = warp + h * kCI_W;
          const int J = b + 1 + (it >> 1), n0 = 16 * (it & 1);
          if (it < nitems && n0 < ci_tw(J, K)) ci_put<0>(T.tile(b, J), ci_tw(J, K), n0, acc[h]);
        }
        __syncthreads();
      }
      CI_STAMP(4 + 2 * b);
      if (b + 1 >= nb) break;
      // ---- trailing update with lookahead: warp 0 updates and factors the
      //      next diagonal tile while the other warps update the rest ----
      if (warp == 0) {
        const int nx = b + 1;
        ci_syrk_item(T, b, nx, nx, 0);
        if (ci_tw(nx, K) > 16) ci_syrk_item(T, b, nx, nx, 16);
        __syncwarp();
        if (ci_diag(T.tile(nx, nx), s_rowbuf, ci_tw(nx, K), nx == nb - 1 ? ci_tw(nx, K) - 1 : -1, pivot_floor) && lane == 0) s_bad = 1;
      } else {
        int it = 0;
        for (int J = b + 1; J < nb; ++J) {
          const int wJ = ci_tw(J, K);
          for (int I = b + 1; I <= J; ++I) {
            if (I == b + 1 && J == b + 1) continue;
            for (int h = 0; h < 2; ++h) {
              const int n0 = 16 * h;
              if (n0 >= wJ) continue;
              if (it++ % (kCI_W - 1) != warp - 1) continue;
              ci_syrk_item(T, b, I, J, n0);
            }
          }
        }
      }
      __syncthreads();
      CI_STAMP(5 + 2 * b);
    }
    if (!s_bad) break;
    if (a.iter == 1 && !shifted) {
      shift = 11.0 * ((double)a.nrows * K + (double)K * (K + 1)) * 2.220446049250313e-16 * tr;
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

  CI_STAMP(40);
  // ---- in-place inverse, row blocks bottom-up ----
  for (int I = nb - 2; I >= 0; --I) {
    const int nitems = (nb - 1 - I) * 2;  // <= 12
    const double* Di = T.tile(I, I);
    double acc[2][4][2][2];
    // W(I, J) = -Dinv_I R(I, J)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int it = warp + h * kCI_W;
      const int J = I + 1 + (it >> 1), n0 = 16 * (it & 1);
      if (it < nitems && n0 < ci_tw(J, K)) {
        const int wJ = ci_tw(J, K);
        const double* tj = T.tile(I, J);
        ci_zero(acc[h]);
        ci_mma(acc[h], n0, [&](int mm, int k) { return Di[k * kCI_LD + mm]; },
               [&](int k, int n) { return n < wJ ? tj[n * kCI_LD + k] : 0.0; });
      }
    }
    __syncthreads();
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int it = warp + h * kCI_W;
      const int J = I + 1 + (it >> 1), n0 = 16 * (it & 1);
      if (it < nitems && n0 < ci_tw(J, K)) ci_put<2>(T.tile(I, J), ci_tw(J, K), n0, acc[h]);
    }
    __syncthreads();
    // Rinv(I, J) = sum_{L=I+1..J} W(I, L) Rinv(L, J)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int it = warp + h * kCI_W;
      const int J = I + 1 + (it >> 1), n0 = 16 * (it & 1);
      if (it < nitems && n0 < ci_tw(J, K)) {
        const int wJ = ci_tw(J, K);
        ci_zero(acc[h]);
        for (int L = I + 1; L <= J; ++L) {
          const int wL = ci_tw(L, K);
          const double* w = T.tile(I, L);
          const double* rl = T.tile(L, J);
          ci_mma(acc[h], n0, [&](int mm, int k) { return k < wL ? w[k * kCI_LD + mm] : 0.0; },
                 [&](int k, int n) { return n < wJ ? rl[n * kCI_LD + k] : 0.0; });
        }
      }
    }
    __syncthreads();
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int it = warp + h * kCI_W;
      const int J = I + 1 + (it >> 1), n0 = 16 * (it & 1);
      if (it < nitems && n0 < ci_tw(J, K)) ci_put<0>(T.tile(I, J), ci_tw(J, K), n0, acc[h]);
    }
    __syncthreads();
  }
  CI_STAMP(41);
  // ---- write dense Rinv (rows by warps; zeros below the diagonal) ----
  for (int gi = warp; gi < K; gi += kCI_W) {
    const int row = a.perm_out ? gperm(gi, K) : gi;
    const int I = gi >> 5, ri = gi & 31;
    double* out = a.Rinv + (size_t)row * K;
    for (int gj = lane; gj < K; gj += 32)
      out[gj] = gj >= gi ? T.tile(I, gj >> 5)[(gj & 31) * kCI_LD + ri] : 0.0;
  }
  __syncthreads();
  CI_STAMP(42);
}

}  // namespace tfk
