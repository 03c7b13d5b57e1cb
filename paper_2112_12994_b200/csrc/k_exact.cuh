// k_exact.cuh -- the reference's rank-revealing solve of one sampled lag
// system (toeplitz.cpp:57-85: Eigen ColPivHouseholderQR with threshold
// tol = max(rows, cols) eps, rank = #{|r_ii| > tol max|r_ii|}; full rank ->
// qr.solve, otherwise BDCSVD's minimum-norm solution with the same threshold),
// for every K, on the GPU:
//
//  1. k_gram_dd + k_gram_dd_reduce: G = A^T A of the gathered, weighted rows
//     A = [X | b] (K = p + 1 columns) in double-double.  Each product is
//     error-free (p = a b, e = fma(a, b, -p)) and the sums are TwoSum
//     accumulated, so G is exact to ~1e-30 relative -- far below the CPQR
//     threshold's square (tol^2 >= 1e-31 only for c < 2, never in practice:
//     tol^2 = (c eps)^2 ~ 5e-24 at c = 1e4).
//  2. k_pchol_dd: diagonally pivoted Cholesky of G in double-double.  In exact
//     arithmetic this is the column-pivoting Householder QR of X: step k picks
//     the column of largest remaining norm (the Schur diagonal, which is
//     Eigen's updated column norm squared) and |r_kk|^2 is that diagonal; the
//     target column rides along unpivoted, so its column of R is z = Q^T b.
//     Rank by Eigen's rule; full rank -> phi by double-double back-substitution.
//  3. k_svd_minnorm (rank-deficient systems only; one thread-block cluster):
//     one-sided block Jacobi on N = [R'^T; z^T] (R' the pivoted p x p factor),
//     so N J = W; then R' = J Sigma U^T with W = U Sigma and the minimum-norm
//     solution x = sum_{s_i >= tol s_max} w_i (J^T z)_i / s_i^2 (BDCSVD's
//     premultiplied threshold, JacobiSVD / BDCSVD _solve_impl semantics).
//
// Why not CholeskyQR here: the BASELINE C4 systems have cond ~ 1e16-1e21, so
// fp64 Gram / preconditioned CholeskyQR factors cannot resolve |r_kk| near the
// threshold (4.4e-11 |r_11| at c = 2e5); shifted CholeskyQR3 breaks down
// (tools/rank_experiment.py).  The double-double Gram keeps the whole
// decision exact at the cost of ~10 fp64 operations per multiply-add.
#pragma once

#include <cooperative_groups.h>

#include "common.cuh"
#include "k_gram.cuh"

namespace tfk {

// ---------------------------------------------------------------- double-double
// Every operation goes through __dadd_rn / __dsub_rn / __dmul_rn: the compiler
// may not contract them into an FMA (which would break the error-free
// transformations -- e.g. s = h + a*b fused into fma(a, b, h) makes TwoSum's
// error term wrong by up to eps |a b|).
struct DD {
  double h, l;
};
__device__ __forceinline__ DD dd_two_sum(double a, double b) {
  const double s = __dadd_rn(a, b);
  const double bb = __dsub_rn(s, a);
  return {s, __dadd_rn(__dsub_rn(a, __dsub_rn(s, bb)), __dsub_rn(b, bb))};
}
__device__ __forceinline__ DD dd_fast(double a, double b) {  // |a| >= |b|
  const double s = __dadd_rn(a, b);
  return {s, __dsub_rn(b, __dsub_rn(s, a))};
}
__device__ __forceinline__ DD dd_add(DD a, DD b) {
  DD s = dd_two_sum(a.h, b.h);
  const DD t = dd_two_sum(a.l, b.l);
  s.l = __dadd_rn(s.l, t.h);
  s = dd_fast(s.h, s.l);
  s.l = __dadd_rn(s.l, t.l);
  return dd_fast(s.h, s.l);
}
__device__ __forceinline__ DD dd_neg(DD a) { return {-a.h, -a.l}; }
__device__ __forceinline__ DD dd_mul(DD a, DD b) {
  const double p = __dmul_rn(a.h, b.h);
  double e = fma(a.h, b.h, -p);
  e = fma(a.h, b.l, e);
  e = fma(a.l, b.h, e);
  return dd_fast(p, e);
}
__device__ __forceinline__ DD dd_div(DD a, DD b) {
  const double q1 = __ddiv_rn(a.h, b.h);
  DD r = dd_add(a, dd_neg(dd_mul(b, DD{q1, 0.0})));
  const double q2 = __ddiv_rn(r.h, b.h);
  r = dd_add(r, dd_neg(dd_mul(b, DD{q2, 0.0})));
  const double q3 = __ddiv_rn(r.h, b.h);
  return dd_add(dd_fast(q1, q2), DD{q3, 0.0});
}
__device__ __forceinline__ DD dd_sqrt(DD a) {
  if (!(a.h > 0.0)) return {0.0, 0.0};
  const double x = __dsqrt_rn(a.h);
  const DD d = dd_add(a, dd_neg(dd_mul(DD{x, 0.0}, DD{x, 0.0})));
  return dd_fast(x, __ddiv_rn(d.h, __dmul_rn(2.0, x)));
}
__device__ __forceinline__ bool dd_gt(DD a, DD b) { return a.h > b.h || (a.h == b.h && a.l > b.l); }
// acc += a * b, exact product, TwoSum into (h, l)
__device__ __forceinline__ void dd_acc(double& h, double& l, double a, double b) {
  const double p = __dmul_rn(a, b);
  const double e = fma(a, b, -p);
  const double s = __dadd_rn(h, p);
  const double bb = __dsub_rn(s, h);
  l = __dadd_rn(l, __dadd_rn(__dadd_rn(__dsub_rn(h, __dsub_rn(s, bb)), __dsub_rn(p, bb)), e));
  h = s;
}
// acc += a * b for double-double a, b (cross terms to first order)
__device__ __forceinline__ void dd_acc2(double& h, double& l, DD a, DD b) {
  const double p = __dmul_rn(a.h, b.h);
  double e = fma(a.h, b.h, -p);
  e = fma(a.h, b.l, e);
  e = fma(a.l, b.h, e);
  const double s = __dadd_rn(h, p);
  const double bb = __dsub_rn(s, h);
  l = __dadd_rn(l, __dadd_rn(__dadd_rn(__dsub_rn(h, __dsub_rn(s, bb)), __dsub_rn(p, bb)), e));
  h = s;
}
__device__ __forceinline__ DD dd_shfl_xor(DD v, int m) {
  return {__shfl_xor_sync(0xffffffffu, v.h, m), __shfl_xor_sync(0xffffffffu, v.l, m)};
}
__device__ __forceinline__ DD dd_warp_sum(DD v) {  // fixed butterfly order
#pragma unroll
  for (int m = 16; m > 0; m >>= 1) v = dd_add(v, dd_shfl_xor(v, m));
  return v;
}

// ---------------------------------------------------------------- 1. Gram
constexpr int kDDThreads = 256;
constexpr int kDDSlab = 16;

struct GramDDPlan {
  int nblk, npair, nsplit;
  int64_t rps;
};

inline GramDDPlan gram_dd_plan(int64_t rows, int K, int sm_count) {
  GramDDPlan g;
  g.nblk = (K + 63) / 64;
  g.npair = g.nblk * (g.nblk + 1) / 2;
  // one wave: 2 resident CTAs per SM (128 registers) -> at most 2 * SMs CTAs
  const int64_t target = 2LL * sm_count;
  int64_t ns = std::max<int64_t>(1, target / g.npair);
  ns = std::max<int64_t>(1, std::min<int64_t>(ns, (rows + 4 * kDDSlab - 1) / (4 * kDDSlab)));
  int64_t rps = (rows + ns - 1) / ns;
  rps = (rps + kDDSlab - 1) / kDDSlab * kDDSlab;
  g.rps = std::max<int64_t>(rps, kDDSlab);
  g.nsplit = (int)((rows + g.rps - 1) / g.rps);
  if (g.nsplit < 1) g.nsplit = 1;
  return g;
}

// Column sums of squares n_j = sum_t a_tj^2 of the gathered rows (fp64; only
// a bound for the Gram's accumulation bias below): partials per (row split,
// 64-column tile), then a fixed-order sum over the splits.
constexpr int kCnRows = 2048;
template <class L>
__global__ void __launch_bounds__(256) k_colnorm2_part(L ld, int64_t rows, int K, const long long* rows_dev,
                                                       double* __restrict__ part) {
  if (rows_dev) rows = min(rows, (int64_t)*rows_dev);
  __shared__ double red[4][64];
  const int tid = threadIdx.x, col = 64 * blockIdx.x + (tid & 63), rg = tid >> 6;
  const int64_t r0 = (int64_t)blockIdx.y * kCnRows, r1 = min(rows, r0 + kCnRows);
  double s = 0.0;
  if (col < K)
    for (int64_t t = r0 + rg; t < r1; t += 4) {
      const double v = ld(t, col);
      s = fma(v, v, s);
    }
  red[rg][tid & 63] = s;
  __syncthreads();
  if (tid < 64 && col < K) part[(int64_t)blockIdx.y * K + col] = (red[0][tid] + red[1][tid]) + (red[2][tid] + red[3][tid]);
}
__global__ void k_colnorm2_sum(const double* __restrict__ part, int nsplit, int K, double* __restrict__ cn) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= K) return;
  double s = 0.0;
  for (int sp = 0; sp < nsplit; ++sp) s += part[(int64_t)sp * K + j];
  cn[j] = s;
}
// accumulation bias of Gram element (i, j): a power of two >= 4 sqrt(n_i n_j)
// (Cauchy-Schwarz bounds every partial sum by sqrt(n_i n_j)), so that
// h = sigma + sum_t a_ti a_tj always satisfies |h| >= |a_ti a_tj| and the
// error-free update of h is FastTwoSum (3 operations instead of TwoSum's 6).
__device__ __forceinline__ double dd_bias(double ni, double nj) {
  const double b = 4.0 * sqrt(ni) * sqrt(nj) * (1.0 + 1e-6);
  if (!(b > 0.0)) return 0x1.0p-1000;
  int e;
  frexp(b, &e);
  return ldexp(1.0, e);  // 2^e > b
}

// Partial double-double Gram of one 64 x 64 tile pair (I <= J) over a row
// range; element (ty + 16 i, tx + 16 j) per thread (conflict-free shared
// reads).  W[(pair * nsplit + split) * 8192 + {0, 4096} + e] = (hi, lo).
template <class L>
__global__ void __launch_bounds__(kDDThreads, 2) k_gram_dd(L ld, int64_t rows, int K, int nblk, int64_t rps, int nsplit,
                                                        double* __restrict__ W, const long long* rows_dev,
                                                        const double* __restrict__ cn) {
  __shared__ double As[kDDSlab][64], Bs[kDDSlab][64];
  int I, J;
  pair_from_index(blockIdx.x, nblk, I, J);
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  if (rows_dev) rows = min(rows, (int64_t)*rows_dev);  // a shard's draw count (row-sharded sweeps)
  const int64_t r0 = (int64_t)blockIdx.y * rps, r1 = min(rows, r0 + rps);
  double h[4][4], l[4][4];
  auto bias_of = [&](int i, int j) {
    const int gi = 64 * I + ty + 16 * i, gj = 64 * J + tx + 16 * j;
    return dd_bias(gi < K ? cn[gi] : 0.0, gj < K ? cn[gj] : 0.0);
  };
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      h[i][j] = bias_of(i, j);
      l[i][j] = 0.0;
    }
  // 16-column groups of the tile that hold columns < K (small K: most of a
  // 64 x 64 tile is zero padding -- skip its products)
  const int ni = min(4, (K - 64 * I + 15) / 16), nj = min(4, (K - 64 * J + 15) / 16);
  double ra[4], rb[4];
  auto load = [&](int64_t t0) {
    const int64_t t = t0 + ty;
    const bool ok = t < r1;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int ca = 64 * I + tx + 16 * q, cb = 64 * J + tx + 16 * q;
      ra[q] = (ok && ca < K) ? ld(t, ca) : 0.0;
      rb[q] = (ok && cb < K) ? ld(t, cb) : 0.0;
    }
  };
  if (r0 < r1) load(r0);
  for (int64_t t0 = r0; t0 < r1; t0 += kDDSlab) {
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      As[ty][tx + 16 * q] = ra[q];
      Bs[ty][tx + 16 * q] = rb[q];
    }
    __syncthreads();
    if (t0 + kDDSlab < r1) load(t0 + kDDSlab);
#pragma unroll 2
    for (int r = 0; r < kDDSlab; ++r) {
      double a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        a[i] = As[r][ty + 16 * i];
        b[i] = Bs[r][tx + 16 * i];
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {  // h += a b with |h| >= |a b|: FastTwoSum + the fma product error
          if (i >= ni || j >= nj) continue;  // 16-column groups past K (CTA-uniform): all zeros
          const double p = __dmul_rn(a[i], b[j]);
          const double e = fma(a[i], b[j], -p);
          const double s = __dadd_rn(h[i][j], p);
          l[i][j] = __dadd_rn(l[i][j], __dadd_rn(__dsub_rn(p, __dsub_rn(s, h[i][j])), e));
          h[i][j] = s;
        }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) {  // fold l into h (|h| >= |l|): keeps |l| <= ulp(h)
        const DD s = dd_fast(h[i][j], l[i][j]);
        h[i][j] = s.h;
        l[i][j] = s.l;
      }
  }
  double* out = W + ((size_t)blockIdx.x * nsplit + blockIdx.y) * 8192;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      // remove the bias: h - sigma is exact (h in [3 sigma / 4, 5 sigma / 4], Sterbenz)
      const DD v = dd_two_sum(__dsub_rn(h[i][j], bias_of(i, j)), l[i][j]);
      const int e = (ty + 16 * i) * 64 + tx + 16 * j;
      out[e] = v.h;
      out[4096 + e] = v.l;
    }
}

// Row-sharded sweeps: the allgathered double-double Gram partials of every
// shard ([world][2][K*K]: hi plane, lo plane) summed in rank order -- exact to
// double-double and identical on every rank (an fp64 allreduce would round).
__global__ void k_dd_sum_ranks(const double* __restrict__ gg, int world, int64_t KK, double* __restrict__ Gh,
                               double* __restrict__ Gl) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= KK) return;
  DD s{0.0, 0.0};
  for (int r = 0; r < world; ++r) s = dd_add(s, DD{gg[(int64_t)r * 2 * KK + e], gg[(int64_t)r * 2 * KK + KK + e]});
  Gh[e] = s.h;
  Gl[e] = s.l;
}

// split partials summed in split order (deterministic) -> full symmetric
// K x K (row-major) hi / lo planes
__global__ void k_gram_dd_reduce(const double* __restrict__ W, int npair, int nsplit, int nblk, int K,
                                 double* __restrict__ Gh, double* __restrict__ Gl, const int* gate) {
  if (gate && *gate == 0) return;
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)npair * 4096) return;
  const int pair = (int)(e >> 12), loc = (int)(e & 4095);
  int I, J;
  pair_from_index(pair, nblk, I, J);
  const int row = 64 * I + (loc >> 6), col = 64 * J + (loc & 63);
  if (row >= K || col >= K) return;
  DD s{0.0, 0.0};
  for (int sp = 0; sp < nsplit; ++sp) {
    const double* w = W + ((size_t)pair * nsplit + sp) * 8192;
    s = dd_add(s, DD{w[loc], w[4096 + loc]});
  }
  Gh[(int64_t)row * K + col] = s.h;
  Gl[(int64_t)row * K + col] = s.l;
  if (I != J) {
    Gh[(int64_t)col * K + row] = s.h;
    Gl[(int64_t)col * K + row] = s.l;
  }
}

// ---------------------------------------------------------------- 2. pivoted Cholesky
constexpr int kPcThreads = 1024;
constexpr int kPcMaxK = 1024;  // K <= kExactMaxP + 1 (static shared memory: 4 double + 1 int arrays)

struct ExactOut {
  double* phi;     // [p] reference order (lag j + 1 at index j)
  double* coefs;   // nullable, packed
  int64_t coef_off;
  double* taus;    // nullable, [lag - 1] = phi[p - 1]
  int* method;     // nullable, [lag - 1] = 0 exact_qr / 1 exact_svd (toeplitz.hpp:49-56)
  int* rank;       // nullable, [lag - 1] = CPQR rank
  int lag;
  int* sweeps;     // nullable, [lag - 1] = Jacobi sweeps of the minimum-norm SVD (0: full rank)
};

struct PcholArgs {
  const double* Gh;
  const double* Gl;
  int K;
  int rev;         // 0: forward rows (target last, column a = lag p - a); 1: target first (column a = lag a)
  int64_t rows;    // sampled rows (tolerance max(rows, p) eps)
  double* Rh;      // workspace K x K: Rh[col * K + i] = r_{i, pos(col)} (by original column)
  double* Rl;
  double* Dh;      // workspace [2][K]: Schur diagonal by original column, double buffered over
  double* Dl;      //   steps (step k reads buffer k & 1, writes the other: no cross-CTA race)
  double* N;       // SVD input (p + 1) x p, column-major: column i = row i of R', row p = z_i
  int* perm;       // [K] pivot position -> original column
  int* svd;        // [0] rank deficient, [1] rank, [2..] sweep convergence flags (zeroed)
  double* tol;     // [0] tol
  ExactOut o;
  const int* gate;
};

__device__ __forceinline__ int exact_phi_index(int col, int p, int rev) { return rev ? col - 1 : p - 1 - col; }

inline int pchol_ctas(int K, int scheme = 0) {
  if (scheme == 1) return K > 256 ? 16 : K > 128 ? 8 : K > 48 ? 4 : 1;
  return K > 256 ? 8 : K > 96 ? 4 : 1;
}

// One thread-block cluster.  Every CTA keeps an identical copy of the pivot
// order and of r_kk (it computes the same argmax from the same global Schur
// diagonal); the positions of row k are split over all warps of the cluster;
// one cluster barrier per step publishes row k and the updated diagonal.
__global__ void __launch_bounds__(kPcThreads) k_pchol_dd(PcholArgs a) {
  namespace cg = cooperative_groups;
  if (a.gate && *a.gate == 0) return;
  cg::cluster_group clu = cg::this_cluster();
  __shared__ int perm[kPcMaxK];
  __shared__ double ch[kPcMaxK], cl[kPcMaxK];  // pivot column: r_{i,k}, i < k (then reused for z')
  __shared__ double rkh[kPcMaxK], rkl[kPcMaxK];
  __shared__ double wv_h[32], wv_l[32];
  __shared__ int wv_i[32];
  __shared__ double cand_h[2][16], cand_l[2][16];  // per-CTA pivot candidates of the cluster, by step parity
  __shared__ int cand_i[2][16];
  __shared__ int s_stop;
  __shared__ double s_x[2];
  const int K = a.K, p = K - 1;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int cta = (int)clu.block_rank(), nct = (int)clu.num_blocks();
  const int gwarp = cta * (kPcThreads / 32) + warp, nwarps = nct * (kPcThreads / 32);
  const int tc = a.rev ? 0 : p;
  for (int pos = tid; pos < K; pos += kPcThreads) perm[pos] = pos == p ? tc : (a.rev ? pos + 1 : pos);
  for (int col = cta * kPcThreads + tid; col < K; col += nct * kPcThreads) {
    a.Dh[col] = a.Gh[(int64_t)col * K + col];
    a.Dl[col] = a.Gl[(int64_t)col * K + col];
    a.Dh[K + col] = a.Dh[col];
    a.Dl[K + col] = a.Dl[col];
  }
  if (tid == 0) s_stop = p;
  __threadfence();
  clu.sync();
  // Eigen's zero-pivot floor: (max column norm * eps)^2 (ColPivHouseholderQR
  // threshold_helper); pivots below it are exact zeros of a rank-deficient X
  double maxd = 0.0;
  for (int pos = 0; pos < p; ++pos) maxd = fmax(maxd, a.Dh[perm[pos]]);
  const double zfloor = maxd * 4.930380657631324e-32;
  for (int k = 0; k < p; ++k) {
    const double* Dch = a.Dh + (k & 1) * K;
    const double* Dcl = a.Dl + (k & 1) * K;
    double* Dnh = a.Dh + ((k + 1) & 1) * K;
    double* Dnl = a.Dl + ((k + 1) & 1) * K;
    // (a) pivot: largest Schur diagonal among positions [k, p), ties -> first.
    // Step 0 scans the diagonal; later steps reduce the per-CTA candidates
    // the previous step's row computation left in every CTA's shared memory
    // (cand[k & 1], written through DSMEM before the cluster barrier).
    {
      if (k == 0) {
        const int pos = k + tid;
        DD v{-INFINITY, 0.0};  // positions past p never win (Schur diagonals may be negative noise)
        int vi = pos;
        if (pos < p) v = DD{Dch[perm[pos]], Dcl[perm[pos]]};
#pragma unroll
        for (int m = 16; m > 0; m >>= 1) {
          const DD o{__shfl_xor_sync(0xffffffffu, v.h, m), __shfl_xor_sync(0xffffffffu, v.l, m)};
          const int oi = __shfl_xor_sync(0xffffffffu, vi, m);
          if (dd_gt(o, v) || (o.h == v.h && o.l == v.l && oi < vi)) {
            v = o;
            vi = oi;
          }
        }
        if (lane == 0) {
          wv_h[warp] = v.h;
          wv_l[warp] = v.l;
          wv_i[warp] = vi;
        }
        __syncthreads();
      }
      if (warp == 0) {  // the 32 warp candidates / the cluster's CTA candidates, same tie rule
        const int cb = k & 1;
        DD b{-INFINITY, 0.0};
        int bi = 0x7fffffff;
        if (k == 0) {
          b = DD{wv_h[lane], wv_l[lane]};
          bi = wv_i[lane];
        } else if (lane < nct) {
          b = DD{cand_h[cb][lane], cand_l[cb][lane]};
          bi = cand_i[cb][lane];
        }
#pragma unroll
        for (int m = 16; m > 0; m >>= 1) {
          const DD o{__shfl_xor_sync(0xffffffffu, b.h, m), __shfl_xor_sync(0xffffffffu, b.l, m)};
          const int oi = __shfl_xor_sync(0xffffffffu, bi, m);
          if (dd_gt(o, b) || (o.h == b.h && o.l == b.l && oi < bi)) {
            b = o;
            bi = oi;
          }
        }
        if (lane == 0) {
        const int tp = perm[k];  // swap positions k <-> bi (identically in every CTA)
        perm[k] = perm[bi];
        perm[bi] = tp;
        if (!(b.h > zfloor)) s_stop = k;
        const DD r = dd_sqrt(b);
        rkh[k] = r.h;
        rkl[k] = r.l;
        }
      }
      __syncthreads();
    }
    if (s_stop == k) break;
    const int ck = perm[k];
    for (int i = tid; i < k; i += kPcThreads) {
      ch[i] = a.Rh[(int64_t)ck * K + i];
      cl[i] = a.Rl[(int64_t)ck * K + i];
    }
    __syncthreads();
    const DD rkk{rkh[k], rkl[k]};
    // (b) row k: r_kj = (G[ck][col_j] - sum_{i<k} r_ik r_ij) / r_kk, one warp per position j;
    // lane 0 also tracks the warp's best updated diagonal (the next pivot's candidates)
    DD wb{-INFINITY, 0.0};
    int wbi = 0x7fffffff;
    for (int j = k + 1 + gwarp; j < K; j += nwarps) {
      const int cj = perm[j];
      const double* rjh = a.Rh + (int64_t)cj * K;
      const double* rjl = a.Rl + (int64_t)cj * K;
      DD g{0.0, 0.0}, dold{0.0, 0.0};
      if (lane == 0) {  // issued before the dot: their latency overlaps it
        g = DD{a.Gh[(int64_t)ck * K + cj], a.Gl[(int64_t)ck * K + cj]};
        if (j < p) dold = DD{Dch[cj], Dcl[cj]};
      }
      double sh = 0.0, sl = 0.0;
      for (int i = lane; i < k; i += 32) dd_acc2(sh, sl, DD{ch[i], cl[i]}, DD{rjh[i], rjl[i]});
      DD s = dd_warp_sum(dd_two_sum(sh, sl));
      if (lane == 0) {
        const DD r = dd_div(dd_add(g, dd_neg(s)), rkk);
        a.Rh[(int64_t)cj * K + k] = r.h;
        a.Rl[(int64_t)cj * K + k] = r.l;
        if (j < p) {
          const DD d = dd_add(dold, dd_neg(dd_mul(r, r)));
          Dnh[cj] = d.h;
          Dnl[cj] = d.l;
          if (dd_gt(d, wb) || (d.h == wb.h && d.l == wb.l && j < wbi)) {
            wb = d;
            wbi = j;
          }
        }
      }
    }
    if (cta == 0 && tid == 0) {
      a.Rh[(int64_t)ck * K + k] = rkk.h;
      a.Rl[(int64_t)ck * K + k] = rkk.l;
    }
    // this CTA's best candidate for step k + 1 -> slot [cta] of cand[(k + 1) & 1] in every CTA
    if (lane == 0) {
      wv_h[warp] = wb.h;
      wv_l[warp] = wb.l;
      wv_i[warp] = wbi;
    }
    __syncthreads();
    if (warp == 0) {
      DD b{wv_h[lane], wv_l[lane]};
      int bi = wv_i[lane];
#pragma unroll
      for (int m = 16; m > 0; m >>= 1) {
        const DD o{__shfl_xor_sync(0xffffffffu, b.h, m), __shfl_xor_sync(0xffffffffu, b.l, m)};
        const int oi = __shfl_xor_sync(0xffffffffu, bi, m);
        if (dd_gt(o, b) || (o.h == b.h && o.l == b.l && oi < bi)) {
          b = o;
          bi = oi;
        }
      }
      if (lane < nct) {  // lane r writes into CTA r
        const int nb = (k + 1) & 1;
        *clu.map_shared_rank(&cand_h[nb][cta], lane) = b.h;
        *clu.map_shared_rank(&cand_l[nb][cta], lane) = b.l;
        *clu.map_shared_rank(&cand_i[nb][cta], lane) = bi;
      }
    }
    clu.sync();  // barrier.cluster arrive.release / wait.acquire: row k, the diagonal and the candidates visible
  }
  const int kend = s_stop;  // rows kend.. are exact zeros
  // rank (Eigen ColPivHouseholderQR::rank with the prescribed threshold)
  const double tol = (double)max(a.rows, (int64_t)p) * 2.220446049250313e-16;
  double mx = 0.0;
  for (int k = 0; k < kend; ++k) mx = fmax(mx, fabs(rkh[k]));
  int rank = 0;
  for (int k = 0; k < kend; ++k) rank += fabs(rkh[k]) > tol * mx;
  if (cta == 0 && tid == 0) {
    a.svd[0] = rank < p ? 1 : 0;
    a.svd[1] = rank;
    a.tol[0] = tol;
    for (int s = 2; s < 66; ++s) a.svd[s] = 0;
    a.svd[66] = kend;  // nonzero rows of R' (rows past it are Eigen's exact zero pivots)
    if (a.o.method) a.o.method[a.o.lag - 1] = rank < p ? 1 : 0;
    if (a.o.rank) a.o.rank[a.o.lag - 1] = rank;
    if (a.o.sweeps) a.o.sweeps[a.o.lag - 1] = 0;
  }
  if (cta == 0)
    for (int pos = tid; pos < K; pos += kPcThreads) a.perm[pos] = perm[pos];
  if (rank < p) {
    // N = [R'^T; z^T], R' (p x p) in pivot order; zero rows past kend
    const int m = p + 1;
    for (int64_t e = cta * kPcThreads + tid; e < (int64_t)m * p; e += (int64_t)nct * kPcThreads) {
      const int i = (int)(e / m), j = (int)(e % m);  // column i of N = row i of R'; entry j
      double v = 0.0;
      if (i < kend) {
        if (j == p) v = a.Rh[(int64_t)tc * K + i];
        else if (j >= i) v = a.Rh[(int64_t)perm[j] * K + i];
      }
      a.N[e] = v;
    }
    return;
  }
  if (cta != 0) return;
  // full rank: R11 x = z (double-double, column-oriented back substitution)
  for (int i = tid; i < p; i += kPcThreads) {
    ch[i] = a.Rh[(int64_t)tc * K + i];
    cl[i] = a.Rl[(int64_t)tc * K + i];
  }
  __syncthreads();
  for (int k = p - 1; k >= 0; --k) {
    if (tid == 0) {
      const DD x = dd_div(DD{ch[k], cl[k]}, DD{rkh[k], rkl[k]});
      s_x[0] = x.h;
      s_x[1] = x.l;
      const int q = exact_phi_index(perm[k], p, a.rev);
      a.o.phi[q] = x.h + x.l;
      if (a.o.coefs) a.o.coefs[a.o.coef_off + q] = x.h + x.l;
      if (a.o.taus && q == p - 1) a.o.taus[a.o.lag - 1] = x.h + x.l;
    }
    __syncthreads();
    const DD x{s_x[0], s_x[1]};
    const int ckk = perm[k];
    for (int i = tid; i < k; i += kPcThreads) {
      const DD z = dd_add(DD{ch[i], cl[i]}, dd_neg(dd_mul(DD{a.Rh[(int64_t)ckk * K + i], a.Rl[(int64_t)ckk * K + i]}, x)));
      ch[i] = z.h;
      cl[i] = z.l;
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------- 3. minimum-norm SVD
constexpr int kSvdThreads = 1024;  // 32 warps: one column pair per warp per sub-round for blocks of <= 32 columns
constexpr int kSvdMaxCta = 16;
constexpr int kSvdMaxSweeps = 60;

struct SvdArgs {
  double* N;       // (p + 1) x p column-major (in place)
  double* sig;     // [p] singular values
  double* xpart;   // [nblk][p]
  const int* perm;
  int* svd;        // [0] needed, [2 + sweep] rotation flags
  const double* tol;
  int p, nblk, bw, rev;
  ExactOut o;
};

inline size_t svd_smem_bytes(int p, int bw) { return sizeof(double) * 2 * (size_t)bw * (p + 1); }

// round-robin (circle method) pair t of round r among n (even) players
__device__ __forceinline__ void rr_pair(int n, int r, int t, int& a, int& b) {
  a = t == 0 ? n - 1 : (r + t) % (n - 1);
  b = (r - t + (n - 1)) % (n - 1);
}

__global__ void __launch_bounds__(kSvdThreads) k_svd_minnorm(SvdArgs a) {
  namespace cg = cooperative_groups;
  if (a.svd[0] == 0) return;  // full rank (uniform over the cluster)
  cg::cluster_group cl = cg::this_cluster();
  extern __shared__ __align__(128) double sm[];
  // columns of N = the kend nonzero rows of R' (rows past kend are exact zero
  // pivots: zero columns, singular value 0 -- dropped); blocks of bw of them
  // Block count from the actual column count (known only here): the critical
  // path of a sweep is ~ncol sub-rounds whatever the block count, but every
  // round costs a block reload and a cluster barrier (few blocks are better
  // for few columns) while a sub-round's fp64 work grows with the block width
  // (many blocks = many SMs are better for many columns); blocks stay within
  // one warp per pair (bw <= 32) and the shared memory (a.bw).  CTAs past
  // nblk / 2 only join the cluster barriers.
  const int p = a.p, m = p + 1;
  const int ncol = a.svd[66];
  const int bcap = min(a.bw, kSvdThreads / 32);
  int nblk = a.nblk;
  {
    // cost model in SM cycles (measured scale, B200): a round = cluster
    // barrier + reload of two bw x m blocks; a sub-round = max(latency of one
    // pair, fp64 work of the CTA's bw pairs at 64 lanes / clock)
    double best = 1e300;
    for (int nb = 2; nb <= a.nblk; nb += 2) {
      const int b = (ncol + nb - 1) / nb;
      if (b > bcap) continue;
      const double sub = (2.0 * b - 1.0) + (nb - 2.0) * b;
      const double cost = (nb - 1.0) * (2000.0 + 0.32 * b * m) + sub * fmax(500.0, b * 7.0 * m / 64.0);
      if (cost < best) {
        best = cost;
        nblk = nb;
      }
    }
  }
  const int bw = max(1, (ncol + nblk - 1) / nblk);
  const int cta = (int)cl.block_rank(), nct = a.nblk / 2;
  const bool active = cta < nblk / 2;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarp = kSvdThreads / 32;
  double* slot[2] = {sm, sm + (size_t)bw * m};
  __shared__ double nrm[2 * (kSvdThreads / 32)];
  int colof[2];
  int sweep = 0;
  for (; sweep < kSvdMaxSweeps; ++sweep) {
    int rotated = 0;
    for (int r = 0; r < nblk - 1; ++r) {
      if (!active) {  // idle CTA: the round's cluster barrier only
        __threadfence();
        cl.sync();
        continue;
      }
      int ba, bb;
      rr_pair(nblk, r, cta, ba, bb);
      colof[0] = ba * bw;
      colof[1] = bb * bw;
      // a block is bw contiguous columns of N: a flat copy (valid columns
      // only, zeros past ncol), 8 loads in flight per thread
      for (int s = 0; s < 2; ++s) {
        const int c0 = colof[s];
        const int nvalid = max(0, min(bw, ncol - c0)) * m, ntot = bw * m;
        const double* src = a.N + (int64_t)c0 * m;
        double* dst = slot[s];
        for (int e0 = 0; e0 < ntot; e0 += 8 * kSvdThreads) {
          double v[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int e = e0 + u * kSvdThreads + tid;
            v[u] = e < nvalid ? src[e] : 0.0;
          }
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int e = e0 + u * kSvdThreads + tid;
            if (e < ntot) dst[e] = v[u];
          }
        }
      }
      __syncthreads();
      // squared norms of the 2 bw local columns (rows < p), kept current
      // through the round by the rotation identities a' = a - t g, b' = b + t g
      for (int e = warp; e < 2 * bw; e += nwarp) {
        const double* xe = slot[e / bw] + (size_t)(e % bw) * m;
        double q = 0.0;
        for (int i = lane; i < p; i += 32) q = fma(xe[i], xe[i], q);
        q = warp_sum(q);
        if (lane == 0) nrm[e] = q;
      }
      __syncthreads();
      // round 0 of a sweep (every block sits in exactly one CTA): all pairs of
      // the 2 bw local columns, so each block's internal pairs run once per
      // sweep; later rounds: the bw x bw cross pairs of the two blocks only
      const int nl = 2 * bw;
      const int nsub = r == 0 ? nl - 1 : bw;
      for (int sr = 0; sr < nsub; ++sr) {
        for (int t = warp; t < bw; t += nwarp) {
          int u, v;
          if (r == 0) {
            rr_pair(nl, sr, t, u, v);
          } else {
            u = t;
            v = bw + (t + sr) % bw;
          }
          const int gu = colof[u / bw] + u % bw, gv = colof[v / bw] + v % bw;
          if (gu >= ncol || gv >= ncol) continue;
          double* xu = slot[u / bw] + (size_t)(u % bw) * m;
          double* xv = slot[v / bw] + (size_t)(v % bw) * m;
          const double al = nrm[u], be = nrm[v];
          double g4[4] = {0.0, 0.0, 0.0, 0.0};  // four chains: the dot's latency, not its length
          int i = lane;
          for (; i + 96 < p; i += 128) {
#pragma unroll
            for (int u = 0; u < 4; ++u) g4[u] = fma(xu[i + 32 * u], xv[i + 32 * u], g4[u]);
          }
          for (; i < p; i += 32) g4[0] = fma(xu[i], xv[i], g4[0]);
          double ga = warp_sum((g4[0] + g4[1]) + (g4[2] + g4[3]));
          if (ga == 0.0 || fabs(ga) <= 2.220446049250313e-16 * sqrt(al * be)) continue;
          // convergence: a sweep whose rotations all have |g| < 1e-7 sqrt(a b) is
          // the last (Jacobi converges quadratically: what it leaves is ~1e-14,
          // far inside the 1e-4 bar on the minimum-norm answers) -- saves the
          // pure check sweep; its small rotations are still applied
          if (fabs(ga) >= 1e-7 * sqrt(al * be)) rotated = 1;
          // rotation angle (Rutishauser): MUFU reciprocal / reciprocal square
          // root + two Newton steps (~1 ulp) instead of IEEE division / sqrt,
          // which dominate the latency of a sub-round
          double tt;
          if (fabs(ga) > 1e-290 && fabs(be - al) < 1e140 * fabs(ga)) {
            const double zeta = (be - al) * fast_rcp(2.0 * ga);
            const double z2 = fma(zeta, zeta, 1.0);
            tt = (zeta >= 0.0 ? 1.0 : -1.0) * fast_rcp(fabs(zeta) + z2 * fast_rsqrt(z2));
          } else {  // subnormal / extreme ratios: the IEEE formulas
            const double zeta = (be - al) / (2.0 * ga);
            tt = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
          }
          const double cs = fast_rsqrt(fma(tt, tt, 1.0)), sn = cs * tt;
          for (int i = lane; i < m; i += 32) {
            const double x = xu[i], y = xv[i];
            xu[i] = cs * x - sn * y;
            xv[i] = sn * x + cs * y;
          }
          double na = al - tt * ga, nb = be + tt * ga;
          if (!(na > 1e-2 * al && nb > 1e-2 * be)) {  // cancellation: recompute from the rotated columns
            __syncwarp();
            double qa = 0.0, qb = 0.0;
            for (int i = lane; i < p; i += 32) {
              qa = fma(xu[i], xu[i], qa);
              qb = fma(xv[i], xv[i], qb);
            }
            na = warp_sum(qa);
            nb = warp_sum(qb);
          }
          if (lane == 0) {
            nrm[u] = na;
            nrm[v] = nb;
          }
        }
        __syncthreads();
      }
      for (int s = 0; s < 2; ++s) {
        const int c0 = colof[s];
        const int nvalid = max(0, min(bw, ncol - c0)) * m;
        double* dst = a.N + (int64_t)c0 * m;
        for (int e = tid; e < nvalid; e += kSvdThreads) dst[e] = slot[s][e];
      }
      __threadfence();
      cl.sync();
    }
    rotated = __syncthreads_or(rotated);
    if (tid == 0 && rotated) atomicOr(&a.svd[2 + sweep], 1);
    __threadfence();
    cl.sync();
    if (*(volatile int*)&a.svd[2 + sweep] == 0) break;
  }
  if (cta == 0 && tid == 0 && a.o.sweeps) a.o.sweeps[a.o.lag - 1] = sweep + 1;
  // singular values, then the solution x = sum_{s_i >= thr} w_i z_i / s_i^2
  for (int c = cta * 2 * bw + warp; c < min(ncol, (cta + 1) * 2 * bw); c += nwarp) {
    double s2 = 0.0;
    for (int i = lane; i < p; i += 32) {
      const double x = a.N[(int64_t)c * m + i];
      s2 = fma(x, x, s2);
    }
    s2 = warp_sum(s2);
    if (lane == 0) a.sig[c] = sqrt(s2);
  }
  __threadfence();
  cl.sync();
  double smax = 0.0;
  for (int c = 0; c < ncol; ++c) smax = fmax(smax, a.sig[c]);
  const double thr = fmax(smax * a.tol[0], 2.2250738585072014e-308);
  // block pair of this CTA: columns [2 bw cta, 2 bw (cta + 1)) -> partial x
  double* xp = a.xpart + (size_t)cta * p;
  for (int j = tid; j < p; j += kSvdThreads) {
    double acc = 0.0;
    for (int c = cta * 2 * bw; c < min(ncol, (cta + 1) * 2 * bw); ++c) {
      const double s = a.sig[c];
      if (!(s >= thr)) continue;
      acc = fma(a.N[(int64_t)c * m + j], a.N[(int64_t)c * m + p] / (s * s), acc);
    }
    xp[j] = acc;
  }
  __threadfence();
  cl.sync();
  if (cta != 0) return;
  for (int j = tid; j < p; j += kSvdThreads) {
    double x = 0.0;
    for (int c = 0; c < nct; ++c) x += a.xpart[(size_t)c * p + j];
    const int q = exact_phi_index(a.perm[j], p, a.rev);
    a.o.phi[q] = x;
    if (a.o.coefs) a.o.coefs[a.o.coef_off + q] = x;
    if (a.o.taus && q == p - 1) a.o.taus[a.o.lag - 1] = x;
  }
}

}  // namespace tfk
