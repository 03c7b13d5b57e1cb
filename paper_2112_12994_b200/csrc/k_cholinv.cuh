// k_cholinv.cuh -- blocked Cholesky factorization G = R^T R of one K x K Gram
// matrix in a single CTA (the small dense core of each CholeskyQR pass that
// replaces Eigen's ColPivHouseholderQR, toeplitz.cpp:57-71).
//
// Output "RD" format (tile-packed upper, k_tpu.cuh): off-diagonal tiles hold
// R, diagonal tiles hold Dinv_J = R_JJ^-1.  No explicit R^-1 is formed:
// consumers apply R^-1 from the right by blocked substitution
// (k_trsm_right), which parallelises over row blocks across CTAs.
//
// For K <= kCholinvMaxK the whole matrix lives in shared memory (207 KB at
// K = 201), moved with cp.async.bulk (TMA engine); larger K work in place on
// a global (L2-resident) copy.  Blocked right-looking, 32-column panels, with
// look-ahead:
//   1. warp 0 factors AND inverts the next diagonal tile (ci_diag32: 8 x 8
//      register blocks + DMMA), overlapped with warps 1..7 finishing the
//      trailing update of the current panel,
//   2. panel row R(b, J) = Dinv_b^T G(b, J)        (DMMA m8n8k4 f64),
//   3. trailing update G(I, J) -= R(b, I)^T R(b, J) (DMMA).
// Breakdown: a non-positive pivot in pass A restarts with the shift
// 11 (cK + K(K+1)) eps tr(G) (shifted CholeskyQR) and flags two extra passes;
// the target (last) pivot is clamped instead (vanishing residual, c == p).
// Pass A also requests pass B when a lower bound of ||R||_F ||R^-1||_F
// exceeds 8 K (CholeskyQR loses orthogonality as cond^2 eps), and always for
// an unpreconditioned system (identity T: first lag, standalone solves).
#pragma once

#ifndef CI_STAMP
#define CI_STAMP(k) ((void)0)
#endif

#include "common.cuh"
#include "k_sample.cuh"
#include "k_tpu.cuh"

namespace tfk {

constexpr int kCholinvMaxK = 203;     // tpu_size(K) * 8 B + 13 KB static <= 227 KB
constexpr int kCholinvThreads = 256;  // 8 warps
constexpr int kCI_W = kCholinvThreads / 32;

__host__ inline size_t cholinv_smem_bytes(int K) { return (size_t)tpu_size(K) * sizeof(double); }
__host__ inline bool cholinv_in_smem(int K) { return K <= kCholinvMaxK; }

struct CholinvArgs {
  const double* G;   // TPU Gram (not modified)
  int K;
  int pass;          // 0 = A (may shift, estimates cond), 1 = B, 2 = C
  int64_t nrows;     // rows of the tall matrix (shift formula)
  double* RD;        // TPU output (RD format); also the working copy when !use_smem
  int use_smem;
  int* flags;        // [0] shifted, [1] failed, [2] need pass B
  const int* gate;   // run only if *gate != 0 (nullable)
  int force_b;       // pass A: always request pass B (unpreconditioned system)
  int invert;        // output R^-1 (TPU) instead of the RD factor
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

// store (MODE 0) or subtract (1) a 32 x 16 accumulator into a tile of width w
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
          else *q -= acc[i][j][e];
        }
      }
}

struct CITiles {
  double* base;
  int K;
  __device__ __forceinline__ double* tile(int I, int J) const { return base + tpu_tile(K, I, J); }
};

// Lane-per-column factor + inverse of a 32 x 32 diagonal tile (one warp):
// lane j keeps column j of the tile in registers, and every lane keeps a
// copy of the running diagonal d[i] = G(i, i) - sum R(k, i)^2.  Step k: every
// lane takes the pivot from its own d[k] (no shuffle; all copies are bitwise
// equal), scales its entry of row k (R(k, j)), row k goes to shared memory
// (its slot in S, column-major (k, j)), and each lane folds R(k, i) R(k, j)
// into its rows i in (k, j] and R(k, i)^2 into d[i] -- broadcast reads.  The
// inverse is right-looking too: once x_l = R^-1(l, j) is known, every row i < l
// accumulates R(i, l) x_l, so x_{l-1} is one multiply away.  Pivot rules:
// the target column `last` is clamped to `floor`, earlier columns break down
// at `badfloor`, columns past `last` are identity padding.  Compile-time
// loops (template recursion) keep v[], d[] in registers, and every lane runs
// the same instruction stream (entries below a lane's diagonal are computed
// and ignored) -- lane-dependent branches would serialise the warp.
template <int K, int I>
struct LUpd {  // i > K: v[i] -= R(K, i) R(K, lane), d[i] -= R(K, i)^2
  static __device__ __forceinline__ void run(double (&v)[32], double (&d)[32], const double* S, double rkj) {
    const double r = S[I * kTLD + K];
    v[I] = fma(-r, rkj, v[I]);
    d[I] = fma(-r, r, d[I]);
    LUpd<K, I + 1>::run(v, d, S, rkj);
  }
};
template <int K>
struct LUpd<K, 32> {
  static __device__ __forceinline__ void run(double (&)[32], double (&)[32], const double*, double) {}
};
template <int K>
struct LFac {
  static __device__ __forceinline__ void run(double (&v)[32], double (&d)[32], double* S, double* invd, int lane,
                                             bool& bad, int last, double floor, double badfloor) {
    double piv = d[K];
    if (K == last) {
      if (!(piv > floor)) piv = floor;  // vanishing residual (c == p)
      bad |= !isfinite(piv);
    } else if (last < 0 || K < last) {
      bad |= !(piv > badfloor) || !isfinite(piv);
    }
    const double inv = fast_rsqrt(piv);
    v[K] = lane == K ? piv * inv : v[K] * inv;  // R(K, lane) (lanes < K: ignored)
    if (lane == K) invd[K] = inv;
    if (lane >= K) S[lane * kTLD + K] = v[K];   // row K of R
    __syncwarp();
    LUpd<K, K + 1>::run(v, d, S, v[K]);
    LFac<K + 1>::run(v, d, S, invd, lane, bad, last, floor, badfloor);
  }
};
template <>
struct LFac<32> {
  static __device__ __forceinline__ void run(double (&)[32], double (&)[32], double*, double*, int, bool&, int,
                                             double, double) {}
};
template <int L, int I>
struct LAcc {  // i < L: acc[i] += R(i, L) x_L
  static __device__ __forceinline__ void run(double (&acc)[32], const double* S, double xl) {
    acc[I] = fma(S[L * kTLD + I], xl, acc[I]);
    LAcc<L, I - 1>::run(acc, S, xl);
  }
};
template <int L>
struct LAcc<L, -1> {
  static __device__ __forceinline__ void run(double (&)[32], const double*, double) {}
};
template <int L>
struct LInv {  // x_L = R^-1(L, lane), then its contributions to the rows above
  static __device__ __forceinline__ void run(double (&v)[32], double (&acc)[32], const double* S, const double* invd,
                                             int lane) {
    const double dl = invd[L];
    const double xl = L == lane ? dl : (L < lane ? -acc[L] * dl : 0.0);
    v[L] = xl;
    LAcc<L, L - 1>::run(acc, S, xl);
    LInv<L - 1>::run(v, acc, S, invd, lane);
  }
};
template <>
struct LInv<-1> {
  static __device__ __forceinline__ void run(double (&)[32], double (&)[32], const double*, const double*, int) {}
};

// tile: the m-column diagonal tile (column-major upper, LD kTLD; columns past
// m are identity padding), factored and replaced by Dinv = R^-1.  S (32 x
// kTLD scratch) receives the rows of R, invd the reciprocal pivots.
__device__ __forceinline__ bool ci_diag_tile(double* tile, int m, int last, double floor, double badfloor,
                                             double* S, double* invd, double* /*unused*/) {
  const int lane = threadIdx.x & 31;
  double v[32], d[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    v[i] = lane < m ? (i <= lane ? tile[lane * kTLD + i] : 0.0) : (i == lane ? 1.0 : 0.0);
    d[i] = i < m ? tile[i * kTLD + i] : 1.0;  // every lane: the diagonal
  }
  __syncwarp();
  bool bad = false;
  LFac<0>::run(v, d, S, invd, lane, bad, last, floor, badfloor);
  __syncwarp();
#pragma unroll
  for (int i = 0; i < 32; ++i) d[i] = 0.0;  // reused: the inverse's row accumulators
  LInv<31>::run(v, d, S, invd, lane);
  if (lane < m) {
#pragma unroll
    for (int i = 0; i < 32; ++i) tile[lane * kTLD + i] = i <= lane ? v[i] : 0.0;
  }
  __syncwarp();
  return bad;
}

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

__global__ void __maxnreg__(255) k_cholinv(CholinvArgs a) {
  extern __shared__ __align__(128) double smem[];
  __shared__ int s_bad;
  __shared__ double s_red[kCI_W];
  __shared__ __align__(16) double s_S[32 * kTLD];  // diagonal-tile scratch (identity padded)
  __shared__ double s_DI[4 * 64], s_TS[4 * 64];
  __shared__ __align__(8) uint64_t s_bar;
  const int K = a.K;
  if (a.gate && *a.gate == 0) return;
  if (a.pass > 0 && a.flags[1] != 0) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nb = (K + 31) / 32;
  const int64_t tsz = tpu_size(K);
  CITiles T;
  T.K = K;
  T.base = a.use_smem ? smem : a.RD;
  CI_STAMP(0);

  double shift = 0.0;
  int shifted = 0;
  double tr = 0.0;
  if (a.use_smem && tid == 0) mbar_init(&s_bar, 1);
  for (int attempt = 0; attempt < 2; ++attempt) {
    if (a.use_smem) {
      if (tid == 0) {  // bulk copy of the TPU image (mbarrier phase = attempt)
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
      for (int64_t e = tid; e < tsz; e += kCholinvThreads) a.RD[e] = a.G[e];
    }
    __syncthreads();
    if (warp == 0) {  // trace (shift, pivot floor, cond estimate), fixed order
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
    const double bad_floor = (double)max(a.nrows, (int64_t)K) * 2.220446049250313e-16 * tr;
    __syncthreads();
    CI_STAMP(1);
    // Iteration b = -1 only factors diagonal tile 0; iteration b applies
    // panel b and, with look-ahead, warp 0 updates + factors diagonal tile
    // b + 1 while warps 1..7 finish the trailing update of panel b.
    for (int b = -1; b < nb && !s_bad; ++b) {
      if (b >= 0) {
        const double* Db = T.tile(b, b);  // Dinv_b
        // panel: R(b, J) = Dinv_b^T G(b, J); items (J, column half) are column-disjoint
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
        CI_STAMP(4 + 3 * b);
      }
      if (b + 1 >= nb) break;
      const int nx = b + 1;
      if (warp == 0) {
        if (b >= 0) {
          ci_syrk_item(T, b, nx, nx, 0);
          if (tpu_w(nx, K) > 16) ci_syrk_item(T, b, nx, nx, 16);
          __syncwarp();
        }
        const int mx = tpu_w(nx, K);
        if (nx == 1) CI_STAMP(60);
        const bool bad = ci_diag_tile(T.tile(nx, nx), mx, nx == nb - 1 ? mx - 1 : -1, pivot_floor, bad_floor,
                                      s_S, s_DI, s_TS);
        if (nx == 1) CI_STAMP(61);
        if (bad && lane == 0) s_bad = 1;
      } else if (b >= 0) {
        int it = 0;
        for (int J = b + 1; J < nb; ++J) {
          const int wJ = tpu_w(J, K);
          for (int I = b + 1; I <= J; ++I) {
            if (I == nx && J == nx) continue;
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
      if (b >= 0) CI_STAMP(5 + 3 * b);
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
  CI_STAMP(41);
  // ---- pass A: cond lower bound ||R||_F^2 = tr(G) + K shift, ||R^-1||_F^2 >= sum ||Dinv_J||_F^2 ----
  if (a.pass == 0) {
    double ss = 0.0;
    for (int J = warp; J < nb; J += kCI_W) {
      const double* dt = T.tile(J, J);
      const int w = tpu_w(J, K);
      for (int e = lane; e < 32 * w; e += 32) {
        const double v = dt[(e >> 5) * kTLD + (e & 31)];
        ss = fma(v, v, ss);
      }
    }
    ss = warp_sum(ss);
    if (lane == 0) s_red[warp] = ss;
    __syncthreads();
    if (tid == 0) {
      double t = 0.0;
      for (int w = 0; w < kCI_W; ++w) t += s_red[w];
      const double cond_lb = sqrt((tr + K * shift) * t);
      a.flags[0] = shifted;
      a.flags[1] = 0;
      a.flags[2] = (a.force_b || shifted || !(cond_lb <= 8.0 * K)) ? 1 : 0;
    }
  }
  // ---- R^-1 in place, block rows bottom-up:
  //      Rinv(I, J) = -Dinv_I sum_{L = I+1..J} R(I, L) Rinv(L, J),  Rinv(J, J) = Dinv_J.
  //      Items (J, column half) run in rounds of 8 with J descending, so a
  //      round only reads R(I, L <= J) tiles that no earlier round overwrote;
  //      products land in registers before the barrier, the writes follow it.
  if (a.invert) {
    for (int I = nb - 2; I >= 0; --I) {
      const int nitems = 2 * (nb - 1 - I);
      for (int r0 = 0; r0 < nitems; r0 += kCI_W) {
        const int it = r0 + warp;
        int J = 0, n0 = 0, wJ = 0;
        bool act = false;
        double acc[4][2][2];
        ci_zero(acc);
        if (it < nitems) {
          J = nb - 1 - (it >> 1);
          n0 = 16 * (it & 1);
          wJ = tpu_w(J, K);
          act = n0 < wJ;
        }
        if (act) {
          for (int L = I + 1; L <= J; ++L) {
            const double* rIL = T.tile(I, L);
            const double* vLJ = T.tile(L, J);
            const int wL = tpu_w(L, K);
            ci_mma(acc, n0, [&](int mm, int k) { return k < wL ? rIL[k * kTLD + mm] : 0.0; },
                   [&](int k, int n) { return (n < wJ && k < wL) ? vLJ[n * kTLD + k] : 0.0; });
          }
        }
        __syncthreads();
        if (act) {
          double* tIJ = T.tile(I, J);
          ci_put<0>(tIJ, wJ, n0, acc);
          __syncwarp();
          const double* dI = T.tile(I, I);
          double acc2[4][2][2];
          ci_zero(acc2);
          ci_mma(acc2, n0, [&](int mm, int k) { return dI[k * kTLD + mm]; },
                 [&](int k, int n) { return n < wJ ? tIJ[n * kTLD + k] : 0.0; });
          __syncwarp();
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 2; ++j) acc2[i][j][0] = -acc2[i][j][0], acc2[i][j][1] = -acc2[i][j][1];
          ci_put<0>(tIJ, wJ, n0, acc2);
        }
        __syncthreads();
      }
    }
  }
  // ---- write RD / R^-1 (TPU) ----
  if (a.use_smem) {
    fence_proxy_async_smem();
    __syncthreads();
    if (tid == 0) {
      const uint32_t bytes = (uint32_t)(tsz * sizeof(double));
      const uint32_t chunk = 32768;
      for (uint32_t off = 0; off < bytes; off += chunk)
        bulk_s2g(reinterpret_cast<char*>(a.RD) + off, reinterpret_cast<const char*>(smem) + off,
                 min(chunk, bytes - off));
      bulk_commit_wait_all();
    }
  }
  CI_STAMP(42);
}

// ---------------------------------------------------------------------------
// X = A Rinv for upper-triangular TPU A and Rinv (S = T R_A^-1, S_B = S_A R_B^-1):
// one CTA per output tile (I <= J), one warp per column half;
// X(I, J) = sum_{L = I..J} A(I, L) Rinv(L, J).  X2 (nullable) gets a copy.
__global__ void __launch_bounds__(64)
    k_trmm_tpu(const double* __restrict__ A, const double* __restrict__ Rinv, double* __restrict__ X,
               double* __restrict__ X2, int K, const int* gate) {
  if (gate && *gate == 0) return;
  const int nb = (K + 31) / 32;
  int rem = blockIdx.x, I = 0;
  while (rem >= nb - I) {
    rem -= nb - I;
    ++I;
  }
  const int J = I + rem;
  const int warp = threadIdx.x >> 5;
  const int n0 = 16 * warp;
  const int wJ = tpu_w(J, K);
  if (n0 >= wJ) return;
  double acc[4][2][2];
  ci_zero(acc);
  for (int L = I; L <= J; ++L) {
    const double* aIL = A + tpu_tile(K, I, L);
    const double* rLJ = Rinv + tpu_tile(K, L, J);
    const int wL = tpu_w(L, K);
    ci_mma(acc, n0, [&](int mm, int k) { return k < wL ? __ldg(aIL + k * kTLD + mm) : 0.0; },
           [&](int k, int n) { return (n < wJ && k < wL) ? __ldg(rLJ + n * kTLD + k) : 0.0; });
  }
  ci_put<0>(X + tpu_tile(K, I, J), wJ, n0, acc);
  if (X2) ci_put<0>(X2 + tpu_tile(K, I, J), wJ, n0, acc);
}

// ---------------------------------------------------------------------------
// X = B R^-1 for R in RD format, by blocked right substitution over tile
// columns: X(:, J) = (B(:, J) - sum_{L<J} X(:, L) R(L, J)) Dinv_J.
// One CTA per 32-row block of B (row blocks are independent); 2 warps
// (column halves); the CTA's row block of X stays in shared memory.
//   dense mode: B, X row-major [rows][ld]           (Q2 = Q1 R_A^-1)
//   tpu mode:   B, X upper-triangular TPU (K x K)   (S = T R_A^-1)
constexpr int kTrsmThreads = 64;

template <bool TPU>
__global__ void __launch_bounds__(kTrsmThreads)
    k_trsm_right(const double* __restrict__ B, const double* __restrict__ RD, double* __restrict__ X,
                 int64_t rows, int K, int64_t ld, const int* gate) {
  if (gate && *gate == 0) return;
  extern __shared__ __align__(16) double xs[];  // tile columns of this row block, [nb][32 cols][kTLD]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nb = (K + 31) / 32;
  const int I = blockIdx.x;  // row block
  const int64_t r0 = (int64_t)I * 32;
  const int jstart = TPU ? I : 0;
  const int n0 = 16 * warp;
  for (int J = jstart; J < nb; ++J) {
    const int wJ = tpu_w(J, K);
    double acc[4][2][2];
    ci_zero(acc);
    double* xj = xs + (size_t)J * 32 * kTLD;
    if (n0 < wJ) {
      for (int L = jstart; L < J; ++L) {
        const int wL = tpu_w(L, K);
        const double* rl = RD + tpu_tile(K, L, J);
        const double* xl = xs + (size_t)L * 32 * kTLD;
        ci_mma(acc, n0, [&](int mm, int k) { return k < wL ? xl[k * kTLD + mm] : 0.0; },
               [&](int k, int n) { return n < wJ ? __ldg(rl + n * kTLD + k) : 0.0; });
      }
      // Y(:, J) = B(:, J) - acc, staged in xs
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int r = 8 * i + (lane >> 2), c = n0 + 8 * j + 2 * (lane & 3) + e;
            if (c < wJ) {
              double bv = 0.0;
              if (TPU) {
                const int gr = 32 * I + r, gc = 32 * J + c;
                if (gr < K && gr <= gc) bv = B[tpu_idx(K, gr, gc)];
              } else if (r0 + r < rows) {
                bv = B[(r0 + r) * ld + 32 * J + c];
              }
              xj[c * kTLD + r] = bv - acc[i][j][e];
            }
          }
    }
    __syncthreads();
    // X(:, J) = Y(:, J) Dinv_J
    if (n0 < wJ) {
      const double* dj = RD + tpu_tile(K, J, J);
      ci_zero(acc);
      ci_mma(acc, n0, [&](int mm, int k) { return k < wJ ? xj[k * kTLD + mm] : 0.0; },
             [&](int k, int n) { return n < wJ ? __ldg(dj + n * kTLD + k) : 0.0; });
    }
    __syncthreads();
    if (n0 < wJ) {
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int r = 8 * i + (lane >> 2), c = n0 + 8 * j + 2 * (lane & 3) + e;
            if (c < wJ) {
              xj[c * kTLD + r] = acc[i][j][e];
              if (TPU) {
                const int gr = 32 * I + r, gc = 32 * J + c;
                if (gr < K && (gr <= gc || (gr >> 5) == (gc >> 5)))
                  X[tpu_idx(K, gr, gc)] = gr <= gc ? acc[i][j][e] : 0.0;
              } else if (r0 + r < rows) {
                X[(r0 + r) * ld + 32 * J + c] = acc[i][j][e];
              }
            }
          }
    }
    __syncthreads();
  }
}

inline size_t trsm_smem_bytes(int K) { return (size_t)((K + 31) / 32) * 32 * kTLD * sizeof(double); }

}  // namespace tfk

namespace tfk {

// ---------------------------------------------------------------------------
// phi straight from the Cholesky factors (RD format) -- O(K^2) per pass, no
// explicit inverse:  S = T R_A^-1 [R_B^-1 [R_C^-1]] is never formed.
//   forward order (target last):  s = S e_last;  phi_fwd = -s[:p] / s[p]
//   reversed order (target first): s0 = S^T e_0, v = S s0 / ||s0||^2,
//                                   phi[j] = -v[1 + j]; rest = 1 / ||s0||^2
// One CTA; 8 threads per row (column) of a 32-block, shuffle-reduced dots.
struct PhiSolveArgs {
  int K;
  const double* T;    // TPU preconditioner
  const double* RA;   // RD factors
  const double* RB;
  const double* RC;
  const int* flags;   // [0] shifted (pass C ran), [1] failed, [2] pass B ran
  int rev;
  double* phi;
  double* coefs;
  int64_t coef_off;
  double* taus;
  int* method;
  int lag;
  double* rest_out;
};

constexpr int kPhiThreads = 256;

__device__ __forceinline__ double oct_sum(double v) {
  v += __shfl_xor_sync(0xffffffffu, v, 1);
  v += __shfl_xor_sync(0xffffffffu, v, 2);
  v += __shfl_xor_sync(0xffffffffu, v, 4);
  return v;
}

// x <- R^-1 x (back substitution, R in RD format), right-looking: once block
// J is final (x_J = Dinv_J x_J, one warp), every warp subtracts R(I, J) x_J
// from a block I < J -- the tile loads of a step are independent (one memory
// round trip per block instead of one per column group)
__device__ void rd_solve_col(const double* R, int K, double* x, double* tmp) {
  (void)tmp;
  const int nb = (K + 31) / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int J = nb - 1; J >= 0; --J) {
    const int wJ = tpu_w(J, K);
    if (warp == 0) {
      const double* D = R + tpu_tile(K, J, J);
      double q0 = 0.0, q1 = 0.0;
      if (lane < wJ) {
#pragma unroll 8
        for (int c = lane; c < wJ; c += 2) {
          q0 = fma(D[c * kTLD + lane], x[32 * J + c], q0);
          if (c + 1 < wJ) q1 = fma(D[(c + 1) * kTLD + lane], x[32 * J + c + 1], q1);
        }
      }
      __syncwarp();
      if (lane < wJ) x[32 * J + lane] = q0 + q1;
    }
    __syncthreads();
    for (int I = warp; I < J; I += nw) {  // blocks above J are full (32 rows)
      const double* Rt = R + tpu_tile(K, I, J);
      double a0 = 0.0, a1 = 0.0;
#pragma unroll 8
      for (int c = 0; c < wJ; c += 2) {
        a0 = fma(Rt[c * kTLD + lane], x[32 * J + c], a0);
        if (c + 1 < wJ) a1 = fma(Rt[(c + 1) * kTLD + lane], x[32 * J + c + 1], a1);
      }
      x[32 * I + lane] -= a0 + a1;
    }
    __syncthreads();
  }
}

// y <- y R^-1 (row vector, forward substitution, R in RD format)
__device__ void rd_solve_row(const double* R, int K, double* y, double* tmp) {
  const int nb = (K + 31) / 32;
  const int c = threadIdx.x >> 3, sub = threadIdx.x & 7;
  for (int J = 0; J < nb; ++J) {
    const int wJ = tpu_w(J, K);
    double part = 0.0;
    if (c < wJ)
      for (int rr = sub; rr < 32 * J; rr += 8)
        part = fma(y[rr], R[tpu_tile(K, rr >> 5, J) + c * kTLD + (rr & 31)], part);
    part = oct_sum(part);
    if (sub == 0 && c < 32) tmp[c] = c < wJ ? y[32 * J + c] - part : 0.0;
    __syncthreads();
    const double* D = R + tpu_tile(K, J, J);
    double q = 0.0;
    if (c < wJ)
      for (int rr = sub; rr <= c; rr += 8) q = fma(tmp[rr], D[c * kTLD + rr], q);
    q = oct_sum(q);
    if (sub == 0 && c < wJ) y[32 * J + c] = q;
    __syncthreads();
  }
}

// s <- T x (upper TPU): a warp per 32-row block I, lane = row, summing the
// tiles T(I, J), J >= I, in order -- coalesced tile columns, loads independent
// across the whole row block
__device__ void tpu_matvec(const double* T, int K, const double* x, double* s) {
  const int nb = (K + 31) / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int I = warp; I < nb; I += nw) {
    const int wI = tpu_w(I, K);
    double a0 = 0.0, a1 = 0.0;
    for (int J = I; J < nb; ++J) {
      const int wJ = tpu_w(J, K);
      const double* Tt = T + tpu_tile(K, I, J);
#pragma unroll 8
      for (int c = 0; c < wJ; c += 2) {
        if (J > I || c >= lane) a0 = fma(__ldg(Tt + c * kTLD + lane), x[32 * J + c], a0);
        if (c + 1 < wJ && (J > I || c + 1 >= lane)) a1 = fma(__ldg(Tt + (c + 1) * kTLD + lane), x[32 * J + c + 1], a1);
      }
    }
    if (lane < wI) s[32 * I + lane] = a0 + a1;
  }
  __syncthreads();
}

__global__ void __launch_bounds__(kPhiThreads) k_phi_solve(PhiSolveArgs a) {
  extern __shared__ double ps[];
  const int K = a.K, p = K - 1;
  const int* fl = a.flags;
  double* x = ps;
  double* s = ps + K;
  double* tmp = ps + 2 * K;
  __shared__ double red[kPhiThreads / 32];
  if (fl[1]) {
    for (int q = threadIdx.x; q < p; q += blockDim.x) a.phi[q] = __longlong_as_double(0x7ff8000000000000ll);
    return;
  }
  const bool hasB = fl[2] != 0, hasC = fl[0] != 0;
  if (!a.rev) {
    for (int i = threadIdx.x; i < K; i += blockDim.x) x[i] = i == p ? 1.0 : 0.0;
    __syncthreads();
    if (hasC) rd_solve_col(a.RC, K, x, tmp);
    if (hasB) rd_solve_col(a.RB, K, x, tmp);
    rd_solve_col(a.RA, K, x, tmp);
    tpu_matvec(a.T, K, x, s);
    const double spp = s[p];
    for (int q = threadIdx.x; q < p; q += blockDim.x) {
      const double v = -s[p - 1 - q] / spp;
      a.phi[q] = v;
      if (a.coefs) a.coefs[a.coef_off + q] = v;
    }
    if (threadIdx.x == 0) {
      if (a.taus) a.taus[a.lag - 1] = -s[0] / spp;
      if (a.method) a.method[a.lag - 1] = hasC ? 3 : (hasB ? 2 : 1);
      if (a.rest_out) a.rest_out[0] = 1.0 / (spp * spp);  // ||r||^2 of this system
    }
    return;
  }
  // reversed: s0 = e_0^T T R_A^-1 R_B^-1 R_C^-1
  for (int i = threadIdx.x; i < K; i += blockDim.x) x[i] = a.T[tpu_idx(K, 0, i)];
  __syncthreads();
  rd_solve_row(a.RA, K, x, tmp);
  if (hasB) rd_solve_row(a.RB, K, x, tmp);
  if (hasC) rd_solve_row(a.RC, K, x, tmp);
  double part = 0.0;
  for (int i = threadIdx.x; i < K; i += blockDim.x) part = fma(x[i], x[i], part);
  part = warp_sum(part);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = part;
  __syncthreads();
  double nrm2 = 0.0;
  for (int w = 0; w < kPhiThreads / 32; ++w) nrm2 += red[w];
  // v = T R_A^-1 R_B^-1 R_C^-1 s0
  if (hasC) rd_solve_col(a.RC, K, x, tmp);
  if (hasB) rd_solve_col(a.RB, K, x, tmp);
  rd_solve_col(a.RA, K, x, tmp);
  tpu_matvec(a.T, K, x, s);
  for (int q = threadIdx.x; q < p; q += blockDim.x) {
    const double v = -s[1 + q] / nrm2;
    a.phi[q] = v;
    if (a.coefs) a.coefs[a.coef_off + q] = v;
    if (a.taus && q == p - 1) a.taus[a.lag - 1] = v;
  }
  if (threadIdx.x == 0) {
    if (a.rest_out) a.rest_out[0] = 1.0 / nrm2;
    if (a.method) a.method[a.lag - 1] = hasC ? 3 : (hasB ? 2 : 1);
  }
}

// First-order inverse of an RD factor, for the NEXT lag's preconditioner only:
// Rinv(J, J) = Dinv_J, Rinv(I, J) ~ -Dinv_I R(I, J) Dinv_J (I < J); the
// neglected terms are O(||Dinv R_off||^2), small because the preconditioned
// Gram is close to the identity.  One CTA per tile pair, one warp per column half.
__global__ void __launch_bounds__(64)
    k_rinv_first_order(const double* __restrict__ RD, double* __restrict__ Ri, int K, const int* gate) {
  if (gate && *gate == 0) return;
  __shared__ double tmp[32 * kTLD];
  const int nb = (K + 31) / 32;
  int rem = blockIdx.x, I = 0;
  while (rem >= nb - I) {
    rem -= nb - I;
    ++I;
  }
  const int J = I + rem;
  const int warp = threadIdx.x >> 5;
  const int n0 = 16 * warp;
  const int wJ = tpu_w(J, K), wI = tpu_w(I, K);
  const double* dJ = RD + tpu_tile(K, J, J);
  double* out = Ri + tpu_tile(K, I, J);
  if (I == J) {
    for (int e = threadIdx.x; e < 32 * wJ; e += 64) {
      const int c = e >> 5, r = e & 31;
      out[c * kTLD + r] = dJ[c * kTLD + r];
    }
    return;
  }
  const double* rIJ = RD + tpu_tile(K, I, J);
  const double* dI = RD + tpu_tile(K, I, I);
  double acc[4][2][2];
  ci_zero(acc);
  if (n0 < wJ)  // tmp = R(I, J) Dinv_J
    ci_mma(acc, n0, [&](int mm, int k) { return k < wJ ? rIJ[k * kTLD + mm] : 0.0; },
           [&](int k, int n) { return (n < wJ && k < wJ) ? dJ[n * kTLD + k] : 0.0; });
  if (n0 < wJ) ci_put<0>(tmp, wJ, n0, acc);
  __syncthreads();
  ci_zero(acc);
  if (n0 < wJ)
    ci_mma(acc, n0, [&](int mm, int k) { return k < wI ? dI[k * kTLD + mm] : 0.0; },
           [&](int k, int n) { return n < wJ ? tmp[n * kTLD + k] : 0.0; });
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) acc[i][j][0] = -acc[i][j][0], acc[i][j][1] = -acc[i][j][1];
  if (n0 < wJ) ci_put<0>(out, wJ, n0, acc);
}

}  // namespace tfk

namespace tfk {

// ---------------------------------------------------------------------------
// Cholesky for K > kCholinvMaxK (the TPU matrix no longer fits one SM's
// shared memory): the same blocked right-looking factorization as k_cholinv,
// one launch per phase of every block step -- the diagonal tile on one CTA,
// the panel and the trailing update spread over many CTAs (2 warps each, one
// per column half) -- on the L2-resident working copy.  Same RD output,
// shift-and-retry on breakdown (pass A), cond gate and flags as k_cholinv.
struct BigChol {
  const double* G;
  double* RD;
  int K;
  int64_t nrows;
  int pass;
  int force_b;
  int* flags;     // solve flags: [0] shifted, [1] failed, [2] need pass B
  int* work;      // [0] bad pivot, [1] attempt armed, [2] shifted
  double* tr;     // trace of G
  const int* gate;
  int* status;
  int lag;
};

__device__ __forceinline__ bool bchol_skip(const BigChol& a) {
  if (a.gate && *a.gate == 0) return true;
  if (a.pass > 0 && a.flags[1] != 0) return true;
  return false;
}

__global__ void k_bchol_arm(BigChol a, int attempt) {
  if (bchol_skip(a) || threadIdx.x != 0) return;
  if (attempt == 0) {
    double t = 0.0;
    for (int i = 0; i < a.K; ++i) t += a.G[tpu_idx(a.K, i, i)];
    a.tr[0] = t;
    a.work[0] = 0;
    a.work[1] = 1;
    a.work[2] = 0;
    return;
  }
  // second attempt only for pass A after a breakdown (shifted CholeskyQR3)
  const int again = a.work[0] != 0 && a.pass == 0;
  if (a.work[0] != 0 && a.pass != 0) {
    a.flags[1] = 1;
    raise_status(a.status, kErrNumerical, a.lag, kReasonCholFail);
  }
  a.work[1] = again;
  if (again) {
    a.work[0] = 0;
    a.work[2] = 1;
  }
}

__global__ void k_bchol_copy(BigChol a) {
  if (bchol_skip(a) || a.work[1] == 0) return;
  const int64_t n = tpu_size(a.K);
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
    a.RD[e] = a.G[e];
}

// shifted retry: RD(i, i) += shift (after the copy kernel)
__global__ void k_bchol_shift(BigChol a) {
  if (bchol_skip(a) || a.work[1] == 0 || a.work[2] == 0) return;
  const double shift = 11.0 * ((double)a.nrows * a.K + (double)a.K * (a.K + 1)) * 2.220446049250313e-16 * a.tr[0];
  for (int i = threadIdx.x; i < a.K; i += blockDim.x) a.RD[tpu_idx(a.K, i, i)] += shift;
}

__global__ void __launch_bounds__(32) k_bchol_diag(BigChol a, int b) {
  if (bchol_skip(a) || a.work[1] == 0 || a.work[0] != 0) return;
  __shared__ __align__(16) double s_S[32 * kTLD];
  __shared__ double s_DI[4 * 64], s_TS[4 * 64];
  const int K = a.K, nb = (K + 31) / 32;
  const int m = tpu_w(b, K);
  const double floor = 4.930380657631324e-32 * a.tr[0];
  const double badfloor = (double)max(a.nrows, (int64_t)K) * 2.220446049250313e-16 * a.tr[0];
  const bool bad =
      ci_diag_tile(a.RD + tpu_tile(K, b, b), m, b == nb - 1 ? m - 1 : -1, floor, badfloor, s_S, s_DI, s_TS);
  if (bad && threadIdx.x == 0) a.work[0] = 1;
}

// R(b, J) = Dinv_b^T G(b, J), J > b: CTA per J, warp per column half
__global__ void __launch_bounds__(64) k_bchol_panel(BigChol a, int b) {
  if (bchol_skip(a) || a.work[1] == 0 || a.work[0] != 0) return;
  const int K = a.K;
  const int J = b + 1 + blockIdx.x;
  const int n0 = 16 * (threadIdx.x >> 5);
  const int wJ = tpu_w(J, K);
  if (n0 >= wJ) return;
  CITiles T;
  T.base = a.RD;
  T.K = K;
  const double* Db = T.tile(b, b);
  double* tj = T.tile(b, J);
  double acc[4][2][2];
  ci_zero(acc);
  ci_mma(acc, n0, [&](int mm, int k) { return Db[mm * kTLD + k]; },
         [&](int k, int n) { return n < wJ ? tj[n * kTLD + k] : 0.0; });
  __syncwarp();
  ci_put<0>(tj, wJ, n0, acc);
}

// G(I, J) -= R(b, I)^T R(b, J) for b < I <= J: CTA per tile pair, warp per column half
__global__ void __launch_bounds__(64) k_bchol_syrk(BigChol a, int b) {
  if (bchol_skip(a) || a.work[1] == 0 || a.work[0] != 0) return;
  const int K = a.K, nb = (K + 31) / 32;
  const int nt = nb - 1 - b;  // trailing tile count
  int rem = blockIdx.x, I = 0;
  while (rem >= nt - I) {
    rem -= nt - I;
    ++I;
  }
  const int J = I + rem;
  const int n0 = 16 * (threadIdx.x >> 5);
  if (n0 >= tpu_w(b + 1 + J, K)) return;
  CITiles T;
  T.base = a.RD;
  T.K = K;
  ci_syrk_item(T, b, b + 1 + I, b + 1 + J, n0);
}

// cond lower bound and the pass flags (as k_cholinv's epilogue)
__global__ void __launch_bounds__(256) k_bchol_finish(BigChol a) {
  if (bchol_skip(a)) return;
  __shared__ double red[8];
  const int K = a.K, nb = (K + 31) / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (a.work[0] != 0) {  // still broken after the retry (or pass B/C breakdown)
    if (threadIdx.x == 0) {
      a.flags[1] = 1;
      raise_status(a.status, kErrNumerical, a.lag, kReasonCholFail);
    }
    return;
  }
  if (a.pass != 0) return;
  double ss = 0.0;
  for (int J = warp; J < nb; J += 8) {
    const double* dt = a.RD + tpu_tile(K, J, J);
    const int w = tpu_w(J, K);
    for (int e = lane; e < 32 * w; e += 32) {
      const double v = dt[(e >> 5) * kTLD + (e & 31)];
      ss = fma(v, v, ss);
    }
  }
  ss = warp_sum(ss);
  if (lane == 0) red[warp] = ss;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < 8; ++w) t += red[w];
    const int shifted = a.work[2];
    const double shift =
        shifted ? 11.0 * ((double)a.nrows * K + (double)K * (K + 1)) * 2.220446049250313e-16 * a.tr[0] : 0.0;
    const double cond_lb = sqrt((a.tr[0] + K * shift) * t);
    a.flags[0] = shifted;
    a.flags[1] = 0;
    a.flags[2] = (a.force_b || shifted || !(cond_lb <= 8.0 * K)) ? 1 : 0;
  }
}

}  // namespace tfk

namespace tfk {

// ---------------------------------------------------------------------------
// Minimum-norm fallback (toeplitz.cpp:72-83 BDCSVD branch): when pass A had
// to shift (a breakdown: the sampled system is rank deficient or nearly so),
// recompute phi as the reference does -- unpivoted Householder QR of the
// c x p system, one-sided Jacobi SVD of R, singular values kept above
// max(c, p) eps s_max, x = sum V_i (R_i^T Q^T b) / s_i^2.  One CTA, the system
// in shared memory (c p <= kMinNormCap); larger degenerate systems keep the
// shifted CholeskyQR3 result (method 3).
constexpr int kMinNormCap = 20000;  // doubles of the c x p system held in shared memory
constexpr int kMinNormThreads = 256;

template <class L>
__global__ void __launch_bounds__(kMinNormThreads)
    k_minnorm(L ld, int64_t c, int K, int rev, int* flags, double* phi, double* coefs, int64_t coef_off,
              double* taus, int* method, int lag, int* status) {
  if (flags[0] == 0) return;  // pass A factored without a breakdown
  const int p = K - 1;
  if (c * (int64_t)p > kMinNormCap || p > 64 || c > 4096) return;
  extern __shared__ double mn[];
  const int rows = (int)c;
  double* M = mn;                     // rows x p, column-major: lag j + 1 in column j
  double* bvec = M + (size_t)rows * p;  // rows
  double* R = bvec + rows;            // p x p (column-major)
  double* V = R + p * p;              // p x p
  __shared__ double red[kMinNormThreads / 32];
  __shared__ double s_beta, s_tau;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = kMinNormThreads / 32;
  for (int e = tid; e < rows * p; e += kMinNormThreads) {
    const int j = e / rows, t = e % rows;
    M[e] = ld(t, rev ? 1 + j : p - 1 - j);
  }
  for (int t = tid; t < rows; t += kMinNormThreads) bvec[t] = ld(t, rev ? 0 : p);
  __syncthreads();
  // Householder QR (LAPACK-style reflectors, as the oracle's restatement)
  const int ksteps = min(rows, p);
  for (int k = 0; k < ksteps; ++k) {
    double* xk = M + (size_t)k * rows + k;
    const int len = rows - k;
    double part = 0.0;
    for (int i = 1 + tid; i < len; i += kMinNormThreads) part = fma(xk[i], xk[i], part);
    part = warp_sum(part);
    if (lane == 0) red[warp] = part;
    __syncthreads();
    if (tid == 0) {
      double tail = 0.0;
      for (int w = 0; w < nw; ++w) tail += red[w];
      const double c0 = xk[0];
      double tau, beta;
      if (tail <= 2.2250738585072014e-308) {
        tau = 0.0;
        beta = c0;
      } else {
        beta = sqrt(c0 * c0 + tail);
        if (c0 >= 0.0) beta = -beta;
        tau = (beta - c0) / beta;
      }
      s_beta = beta;
      s_tau = tau;
    }
    __syncthreads();
    const double beta = s_beta, tau = s_tau;
    const double d = xk[0] - beta;
    if (tau != 0.0)
      for (int i = 1 + tid; i < len; i += kMinNormThreads) xk[i] /= d;
    else
      for (int i = 1 + tid; i < len; i += kMinNormThreads) xk[i] = 0.0;
    __syncthreads();
    if (tid == 0) xk[0] = beta;
    // apply H = I - tau v v^T (v = [1, xk[1..]]) to columns k+1.. and b: one warp per column
    for (int j = k + 1 + warp; j <= p; j += nw) {
      double* cj = j < p ? M + (size_t)j * rows + k : bvec + k;
      double dot = 0.0;
      for (int i = 1 + lane; i < len; i += 32) dot = fma(xk[i], cj[i], dot);
      dot = warp_sum(dot) + cj[0];
      const double f = tau * dot;
      if (lane == 0) cj[0] -= f;
      for (int i = 1 + lane; i < len; i += 32) cj[i] = fma(-f, xk[i], cj[i]);
    }
    __syncthreads();
  }
  // R (upper, p x p; rows >= p here since c >= p_bar >= p) and V = I
  for (int e = tid; e < p * p; e += kMinNormThreads) {
    const int j = e / p, i = e % p;
    R[e] = i <= j ? M[(size_t)j * rows + i] : 0.0;
    V[e] = i == j ? 1.0 : 0.0;
  }
  __syncthreads();
  // one-sided Jacobi on the columns of R, cyclic pair order, one warp (the
  // degenerate path is rare; p <= 64)
  const double eps = 2.220446049250313e-16;
  if (warp == 0) {
    for (int sweep = 0; sweep < 60; ++sweep) {
      bool rotated = false;
      for (int i = 0; i < p - 1; ++i) {
        for (int j = i + 1; j < p; ++j) {
          double a = 0.0, b = 0.0, g = 0.0;
          for (int r = lane; r < p; r += 32) {
            const double ri = R[i * p + r], rj = R[j * p + r];
            a = fma(ri, ri, a);
            b = fma(rj, rj, b);
            g = fma(ri, rj, g);
          }
          a = warp_sum(a);
          b = warp_sum(b);
          g = warp_sum(g);
          if (g != 0.0 && fabs(g) > eps * sqrt(a * b)) {
            const double zeta = (b - a) / (2.0 * g);
            const double tt = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
            const double cs = 1.0 / sqrt(1.0 + tt * tt), sn = cs * tt;
            for (int r = lane; r < p; r += 32) {
              const double ri = R[i * p + r], rj = R[j * p + r];
              R[i * p + r] = cs * ri - sn * rj;
              R[j * p + r] = sn * ri + cs * rj;
              const double vi = V[i * p + r], vj = V[j * p + r];
              V[i * p + r] = cs * vi - sn * vj;
              V[j * p + r] = sn * vi + cs * vj;
            }
            rotated = true;
          }
          __syncwarp();
        }
      }
      if (!rotated) break;
    }
  }
  __syncthreads();
  // x = sum_i V_i (R_i^T qb) / s_i^2 over s_i >= s_max max(c, p) eps
  double* qb = bvec;  // Q^T b: first p entries
  __shared__ double sv[64], coef[64];
  if (tid < p) {
    double s2 = 0.0, dq = 0.0;
    for (int r = 0; r < p; ++r) {
      s2 = fma(R[tid * p + r], R[tid * p + r], s2);
      dq = fma(R[tid * p + r], qb[r], dq);
    }
    sv[tid] = sqrt(s2);
    coef[tid] = s2 > 0.0 ? dq / s2 : 0.0;
  }
  __syncthreads();
  double smax = 0.0;
  for (int i = 0; i < p; ++i) smax = fmax(smax, sv[i]);
  double pre = smax * (double)max((int64_t)p, c) * eps;
  if (pre < 2.2250738585072014e-308) pre = 2.2250738585072014e-308;
  if (tid < p) {
    double x = 0.0;
    for (int i = 0; i < p; ++i)
      if (sv[i] >= pre) x = fma(coef[i], V[i * p + tid], x);
    phi[tid] = x;
    if (coefs) coefs[coef_off + tid] = x;
    if (taus && tid == p - 1) taus[lag - 1] = x;
  }
  if (tid == 0) {
    if (method) method[lag - 1] = 4;  // minimum-norm SVD path
    // a pass B / C breakdown of this lag is answered by the minimum-norm solve
    if (flags[1] != 0 && status[0] == kErrNumerical && status[1] == lag && status[2] == kReasonCholFail)
      status[0] = 0;
    flags[1] = 0;
  }
}

}  // namespace tfk
