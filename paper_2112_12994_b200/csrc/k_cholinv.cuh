// k_cholinv.cuh -- fused Cholesky factorization + triangular inverse of one
// K x K Gram matrix in a single CTA: G = R^T R (upper R), Rinv = R^-1.
//
// This is the small dense core of each CholeskyQR pass that replaces Eigen's
// ColPivHouseholderQR (toeplitz.cpp:57-71) on the sampled system.  Input and
// output are tile-packed upper matrices (k_tpu.cuh); for K <= kCholinvMaxK
// the whole matrix lives in shared memory (207 KB at K = 201), moved in and
// out with cp.async.bulk (TMA engine); larger K work in place in global
// memory (L2-resident).
//
// Blocked right-looking Cholesky, block 32, with look-ahead:
//   * warp 0 updates the next diagonal tile first, then factors and inverts
//     it in registers (lane l owns column l; fully unrolled, __noinline__ so
//     the ~3k-instruction body is fetched once) while warps 1..7 apply the
//     rest of the trailing update;
//   * panel:    R(b, J)  = Dinv_b^T G(b, J)            (DMMA m8n8k4 f64)
//   * trailing: G(I, J) -= R(b, I)^T R(b, J)           (DMMA)
// In-place blocked inverse, row blocks bottom-up:
//   W(I, L)    = -Dinv_I R(I, L)                        (DMMA)
//   Rinv(I, J) = sum_{L=I+1..J} W(I, L) Rinv(L, J)       (DMMA)
// Breakdown handling: a non-positive pivot in pass A restarts with the
// shift 11 (cK + K(K+1)) eps tr(G) (shifted CholeskyQR) and flags the two
// extra passes; the target (last) pivot is clamped instead (c == p case).
// Pass A also estimates cond(R) <= ||R||_F ||R^-1||_F and requests pass B
// when it exceeds 16 K (CholeskyQR loses orthogonality as cond^2 eps).
#pragma once

#ifndef CI_STAMP
#define CI_STAMP(k) ((void)0)
#endif

#include "common.cuh"
#include "k_sample.cuh"
#include "k_tpu.cuh"

namespace tfk {

constexpr int kCholinvMaxK = 211;     // tpu_size(K) * 8 B <= 227 KB - static smem
constexpr int kCholinvThreads = 256;  // 8 warps: warp 0 diagonal chain, 1..7 bulk updates
constexpr int kCI_W = kCholinvThreads / 32;

__host__ inline size_t cholinv_smem_bytes(int K) { return (size_t)tpu_size(K) * sizeof(double); }
__host__ inline bool cholinv_in_smem(int K) { return K <= kCholinvMaxK; }

struct CholinvArgs {
  const double* G;   // TPU Gram (not modified)
  int K;
  int pass;          // 0 = A (may shift, estimates cond), 1 = B, 2 = C
  int64_t nrows;     // rows of the tall matrix (shift formula)
  double* Rinv;      // TPU output; also the working copy when !use_smem
  int use_smem;
  int* flags;        // [0] shifted, [1] failed, [2] need pass B
  const int* gate;   // run only if *gate != 0 (nullable)
  double* scratch;   // global scratch, (K/32) * 32 * 36 doubles (large K only)
  int* status;
  int lag;
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

// store (MODE 0), subtract (1) or store negated (2) a 32 x 16 accumulator
template <int MODE>
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
          double* q = t + c * kTLD + r;
          if (MODE == 0) *q = acc[i][j][e];
          else if (MODE == 1) *q -= acc[i][j][e];
          else *q = -acc[i][j][e];
        }
      }
}

// ---- 32 x 32 diagonal block: factor, then invert in place (one warp) ----
// Lane l owns column l.  A "rotating" register window keeps the row being
// eliminated at d[0] (the window shifts by one row per step), so every step
// is the same compact, fully unrolled body with only compile-time register
// indices: a fully unrolled 32-step version is ~7k instructions, which does
// not stay in the instruction cache between calls.  It is inlined at a single
// call site in uniform control flow so the shuffles compile to plain SHFL
// (a non-inlined callee gets divergence-safe collective sequences, ~10x
// slower).  Finalized rows go to the
// tile in shared memory; the inverse reads row i of R from there (broadcast)
// and keeps the already-computed rows of its column of R^-1 in a window too.
__device__ __forceinline__ bool ci_diag(double* dt, int m, int last, double floor) {
  const int lane = threadIdx.x & 31;
  double* col = dt + lane * kTLD;  // column `lane` (column-major tile)
  double d[32];                    // d[k] = current entry of row (i + k) of my column
#pragma unroll
  for (int k = 0; k < 32; ++k) d[k] = (lane < m && k <= lane) ? col[k] : 0.0;
  bool bad = false;
  for (int i = 0; i < m; ++i) {
    double piv = __shfl_sync(0xffffffffu, d[0], i);
    if (i == last && !(piv > floor)) piv = floor;  // vanishing residual (c == p)
    bad |= !(piv > 0.0) || !isfinite(piv);
    const double inv = fast_rsqrt(piv);
    const double ri = lane == i ? piv * inv : (lane > i ? d[0] * inv : 0.0);  // R(i, lane)
    if (lane >= i && lane < m) col[i] = ri;
#pragma unroll
    for (int k = 1; k < 32; ++k) {
      const double rik = __shfl_sync(0xffffffffu, ri, (i + k) & 31);  // R(i, i + k)
      if (lane >= i + k) d[k] = fma(-rik, ri, d[k]);
    }
#pragma unroll
    for (int k = 0; k < 31; ++k) d[k] = d[k + 1];
    d[31] = 0.0;
  }
  __syncwarp();
  // inverse, rows bottom-up: x(i,l) = (delta_il - sum_{q>i} R(i,q) x(q,l)) / R(i,i);
  // xw[k] = x(i + 1 + k, lane) (zero beyond the column), row i of R read
  // from the tile (broadcast) before row i is overwritten by row i of R^-1
  double xw[32];
#pragma unroll
  for (int k = 0; k < 32; ++k) xw[k] = 0.0;
  for (int i = m - 1; i >= 0; --i) {
    double a0 = (lane == i) ? 1.0 : 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll
    for (int k = 0; k < 31; k += 4) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int q = i + 1 + k + u;
        if (k + u < 31 && q < m) {
          const double rq = dt[q * kTLD + i];  // R(i, q), same address for all lanes
          const double t = xw[k + u];
          if (u == 0) a0 = fma(-rq, t, a0);
          else if (u == 1) a1 = fma(-rq, t, a1);
          else if (u == 2) a2 = fma(-rq, t, a2);
          else a3 = fma(-rq, t, a3);
        }
      }
    }
    const double rinv = fast_rcp(dt[i * kTLD + i]);
    const double xi = lane >= i ? ((a0 + a1) + (a2 + a3)) * rinv : 0.0;
    __syncwarp();
    if (lane >= i && lane < m) col[i] = xi;
#pragma unroll
    for (int k = 31; k > 0; --k) xw[k] = xw[k - 1];
    xw[0] = xi;
    __syncwarp();
  }
  if (lane < m)
    for (int r = lane + 1; r < 32; ++r) col[r] = 0.0;  // strictly lower part
  return __any_sync(0xffffffffu, bad);
}

struct CITiles {
  double* base;
  int K;
  __device__ __forceinline__ double* tile(int I, int J) const { return base + tpu_tile(K, I, J); }
};

__device__ __forceinline__ void ci_syrk_item(const CITiles& T, int b, int I, int J, int n0) {
  const int K = T.K;
  const int wI = tpu_w(I, K), wJ = tpu_w(J, K);
  const double* pI = T.tile(b, I);
  const double* pJ = T.tile(b, J);
  double acc[4][2][2];
  ci_zero(acc);
  ci_mma(acc, n0, [&](int mm, int k) { return mm < wI ? pI[mm * kTLD + k] : 0.0; },
         [&](int k, int n) { return n < wJ ? pJ[n * kTLD + k] : 0.0; });
  ci_put<1>(T.tile(I, J), wJ, n0, acc);
}

__global__ void __launch_bounds__(kCholinvThreads) k_cholinv(CholinvArgs a) {
  extern __shared__ __align__(128) double smem[];
  __shared__ int s_bad;
  __shared__ double s_red[kCI_W];
  __shared__ __align__(8) uint64_t s_bar;
  const int K = a.K;
  if (a.gate && *a.gate == 0) return;
  if (a.pass > 0 && a.flags[1] != 0) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nb = (K + 31) / 32;
  const int64_t tsz = tpu_size(K);
  CITiles T;
  T.K = K;
  T.base = a.use_smem ? smem : a.Rinv;
  CI_STAMP(0);

  double shift = 0.0;
  int shifted = 0;
  double tr = 0.0;
  if (a.use_smem && tid == 0) mbar_init(&s_bar, 1);
  for (int attempt = 0; attempt < 2; ++attempt) {
    if (a.use_smem) {
      // ---- bulk copy of the TPU image into shared memory (phase = attempt) ----
      if (tid == 0) {
        const uint32_t bytes = (uint32_t)(tsz * sizeof(double));
        mbar_expect_tx(&s_bar, bytes);
        const uint32_t chunk = 32768;
        for (uint32_t off = 0; off < bytes; off += chunk)
          bulk_g2s(reinterpret_cast<char*>(smem) + off, reinterpret_cast<const char*>(a.G) + off,
                   min(chunk, bytes - off), &s_bar);
      }
      __syncthreads();
      mbar_wait(&s_bar, (uint32_t)attempt);
    } else {
      // large K: work on a global (L2-resident) copy
      for (int64_t e = tid; e < tsz; e += kCholinvThreads) a.Rinv[e] = a.G[e];
      __threadfence_block();
    }
    __syncthreads();
    // trace (shift, pivot floor, cond estimate) in a fixed order
    if (warp == 0) {
      double t = 0.0;
      for (int i = lane; i < K; i += 32) t += T.base[tpu_idx(K, i, i)];
      t = warp_sum(t);
      if (lane == 0) {
        s_red[0] = t;
        s_bad = 0;
      }
    }
    __syncthreads();
    tr = s_red[0];
    if (attempt > 0)
      for (int i = tid; i < K; i += kCholinvThreads) T.base[tpu_idx(K, i, i)] += shift;
    const double pivot_floor = 4.930380657631324e-32 * tr;  // eps^2 tr(G)
    __syncthreads();
    CI_STAMP(1);
    // Iteration b = -1 only factors the first diagonal tile; iteration b
    // applies panel b and, with look-ahead, factors diagonal tile b + 1 (warp
    // 0) while warps 1..7 finish the trailing update of panel b.
    for (int b = -1; b < nb && !s_bad; ++b) {
      if (b >= 0) {
        const double* Db = T.tile(b, b);
        // ---- panel: R(b, J) = Dinv_b^T G(b, J), J > b.  Items (J, column half)
        //      read and write disjoint columns, so each is updated in place. ----
        const int nitems = (nb - 1 - b) * 2;
        for (int it = warp; it < nitems; it += kCI_W) {
          const int J = b + 1 + (it >> 1), n0 = 16 * (it & 1);
          const int wJ = tpu_w(J, K);
          if (n0 >= wJ) continue;
          double* tj = T.tile(b, J);
          double acc[4][2][2];
          ci_zero(acc);
          ci_mma(acc, n0, [&](int mm, int k) { return Db[mm * kTLD + k]; },
                 [&](int k, int n) { return n < wJ ? tj[n * kTLD + k] : 0.0; });
          __syncwarp();
          ci_put<0>(tj, wJ, n0, acc);
        }
        __syncthreads();
        CI_STAMP(4 + 2 * b);
      }
      if (b + 1 >= nb) break;
      const int nx = b + 1;
      if (warp == 0) {
        if (b >= 0) {
          ci_syrk_item(T, b, nx, nx, 0);
          if (tpu_w(nx, K) > 16) ci_syrk_item(T, b, nx, nx, 16);
          __syncwarp();
        }
        const bool bad = ci_diag(T.tile(nx, nx), tpu_w(nx, K), nx == nb - 1 ? tpu_w(nx, K) - 1 : -1,
                                 pivot_floor);
        if (bad && lane == 0) s_bad = 1;
      } else if (b >= 0) {
        int it = 0;
        for (int J = b + 1; J < nb; ++J) {
          const int wJ = tpu_w(J, K);
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
      if (b >= 0) CI_STAMP(5 + 2 * b);
    }
    if (!s_bad) break;
    if (a.pass == 0 && !shifted) {
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
  CI_STAMP(40);

  // ---- in-place inverse, row blocks bottom-up ----
  for (int I = nb - 2; I >= 0; --I) {
    const int nitems = (nb - 1 - I) * 2;
    const double* Di = T.tile(I, I);
    // W(I, J) = -Dinv_I R(I, J): column-disjoint items, in place
    for (int it = warp; it < nitems; it += kCI_W) {
      const int J = I + 1 + (it >> 1), n0 = 16 * (it & 1);
      const int wJ = tpu_w(J, K);
      if (n0 >= wJ) continue;
      double* tj = T.tile(I, J);
      double acc[4][2][2];
      ci_zero(acc);
      ci_mma(acc, n0, [&](int mm, int k) { return Di[k * kTLD + mm]; },
             [&](int k, int n) { return n < wJ ? tj[n * kTLD + k] : 0.0; });
      __syncwarp();
      ci_put<2>(tj, wJ, n0, acc);
    }
    __syncthreads();
    // Rinv(I, J) = sum_{L=I+1..J} W(I, L) Rinv(L, J): reads all of row I, so
    // every item is computed before any is written (registers, <= 2 per warp,
    // or the global scratch row for large K)
    auto item_rinv = [&](int it, double (&acc)[4][2][2]) {
      const int J = I + 1 + (it >> 1), n0 = 16 * (it & 1);
      const int wJ = tpu_w(J, K);
      ci_zero(acc);
      for (int L = I + 1; L <= J; ++L) {
        const int wL = tpu_w(L, K);
        const double* w = T.tile(I, L);
        const double* rl = T.tile(L, J);
        ci_mma(acc, n0, [&](int mm, int k) { return k < wL ? w[k * kTLD + mm] : 0.0; },
               [&](int k, int n) { return n < wJ ? rl[n * kTLD + k] : 0.0; });
      }
    };
    if (nitems <= 2 * kCI_W) {
      double acc[2][4][2][2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int it = warp + h * kCI_W;
        if (it < nitems && 16 * (it & 1) < tpu_w(I + 1 + (it >> 1), K)) item_rinv(it, acc[h]);
      }
      __syncthreads();
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int it = warp + h * kCI_W;
        const int J = I + 1 + (it >> 1), n0 = 16 * (it & 1);
        if (it < nitems && n0 < tpu_w(J, K)) ci_put<0>(T.tile(I, J), tpu_w(J, K), n0, acc[h]);
      }
    } else {
      for (int it = warp; it < nitems; it += kCI_W) {
        const int J = I + 1 + (it >> 1), n0 = 16 * (it & 1);
        if (n0 >= tpu_w(J, K)) continue;
        double acc[4][2][2];
        item_rinv(it, acc);
        ci_put<0>(a.scratch + (size_t)(J - I - 1) * 32 * kTLD, tpu_w(J, K), n0, acc);
      }
      __syncthreads();
      for (int it = warp; it < nitems; it += kCI_W) {
        const int J = I + 1 + (it >> 1), n0 = 16 * (it & 1);
        const int wJ = tpu_w(J, K);
        if (n0 >= wJ) continue;
        const double* src = a.scratch + (size_t)(J - I - 1) * 32 * kTLD;
        double* dst = T.tile(I, J);
        for (int e = lane; e < 16 * 32; e += 32) {
          const int c = n0 + (e >> 5), r = e & 31;
          if (c < wJ) dst[c * kTLD + r] = src[c * kTLD + r];
        }
      }
    }
    __syncthreads();
  }
  CI_STAMP(41);

  // ---- cond(R) estimate (pass A): ||R||_F^2 = tr(G) + K shift; ||Rinv||_F^2 ----
  if (a.pass == 0) {
    double ss = 0.0;
    for (int64_t e = tid; e < tsz; e += kCholinvThreads) {
      const double v = T.base[e];
      ss = fma(v, v, ss);
    }
    ss = warp_sum(ss);
    if (lane == 0) s_red[warp] = ss;
    __syncthreads();
    if (tid == 0) {
      double t = 0.0;
      for (int w = 0; w < kCI_W; ++w) t += s_red[w];
      const double cond_f = sqrt((tr + K * shift) * t);
      a.flags[0] = shifted;
      a.flags[1] = 0;
      a.flags[2] = (shifted || !(cond_f <= 16.0 * K)) ? 1 : 0;
    }
  }
  // ---- write Rinv (TPU) ----
  if (a.use_smem) {
    fence_proxy_async_smem();
    __syncthreads();
    if (tid == 0) {
      const uint32_t bytes = (uint32_t)(tsz * sizeof(double));
      const uint32_t chunk = 32768;
      for (uint32_t off = 0; off < bytes; off += chunk)
        bulk_s2g(reinterpret_cast<char*>(a.Rinv) + off, reinterpret_cast<const char*>(smem) + off,
                 min(chunk, bytes - off));
      bulk_commit_wait_all();
    }
  }
  CI_STAMP(42);
}

}  // namespace tfk
