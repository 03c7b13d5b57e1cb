// k_gram.cuh -- fp64 tensor-core (DMMA m8n8k4) Gram and Q-formation kernels
// for the CholeskyQR2 solve of the sampled least-squares system
// (replaces the Eigen ColPivHouseholderQR call of toeplitz.cpp:57-71, fed by
// apply_sample, sketch.cpp:61-79).
//
// The sampled, weighted rows are never materialised as a separate matrix:
// row t of the augmented system in forward column order (k_tpu.cuh) is
//   a_t[a] = w_t * y[off + i_t + a],  a = 0..K-1   (K = p + 1, target last)
// a contiguous slice of the series -- the gather is fused into the tile
// loads (apply_sample's product w * y is formed exactly as the reference).
//
//   k_gram   : split-K partial Gram tiles (64x64 upper block pairs) from rows
//              [split * rps, (split+1) * rps); 4 warps, 32x32 per warp,
//              16 DMMA per k4-step.  Deterministic: the last CTA of a tile
//              pair reduces the split partials in split order.
//   k_qform  : Q = A * B for an upper-triangular TPU right factor B
//              (CholeskyQR's Q = A R^-1 and the preconditioned Q1 = A T).
#pragma once

#include "common.cuh"
#include "k_tpu.cuh"

namespace tfk {

struct DenseRows {
  const double* q;
  int64_t ld;
  __device__ __forceinline__ double operator()(int64_t t, int col) const {
    return q[t * ld + col];
  }
};

constexpr int kGramThreads = 128;
constexpr int kSJ = 68;  // padded row stride (doubles): conflict-free fragment loads

__device__ __forceinline__ void pair_from_index(int pair, int nblk, int& jb, int& lb) {
  int rem = pair;
  jb = 0;
  while (rem >= nblk - jb) {
    rem -= nblk - jb;
    ++jb;
  }
  lb = jb + rem;
}

// Split-K partial tiles go to W; the last CTA of each tile pair (arrival
// counted with an atomic ticket) sums the partials in split order and writes
// G -- deterministic, and no separate reduction launch.
template <class L>
__global__ void __launch_bounds__(kGramThreads)
    k_gram(L ld, int64_t rows, int K, int nblk, int64_t rows_per_split, double* __restrict__ W,
           double* __restrict__ G, int* __restrict__ tickets, const int* skip_flag) {
  if (skip_flag && *skip_flag == 0) return;
  __shared__ __align__(16) double SJ[32][kSJ];
  __shared__ __align__(16) double SL[32][kSJ];
  int jb, lb;
  pair_from_index(blockIdx.x, nblk, jb, lb);
  const bool diag = jb == lb;
  const int J0 = jb * 64, L0 = lb * 64;
  const int64_t rb = (int64_t)blockIdx.y * rows_per_split;
  const int64_t re = min(rows, rb + rows_per_split);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp & 1, wn = warp >> 1;
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  const int cc = tid & 63, rsub = tid >> 6;
  for (int64_t r0 = rb; r0 < re; r0 += 32) {
#pragma unroll 4
    for (int s = 0; s < 16; ++s) {
      const int rr = rsub + 2 * s;
      const int64_t row = r0 + rr;
      double vj = 0.0, vl = 0.0;
      if (row < re) {
        if (J0 + cc < K) vj = ld(row, J0 + cc);
        if (!diag && L0 + cc < K) vl = ld(row, L0 + cc);
      }
      SJ[rr][cc] = vj;
      SL[rr][cc] = vl;
    }
    __syncthreads();
    const double(*B)[kSJ] = diag ? SJ : SL;
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      const int tr = 4 * kk + (lane & 3);
      double af[4], bf[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) af[i] = SJ[tr][32 * wm + 8 * i + (lane >> 2)];
#pragma unroll
      for (int j = 0; j < 4; ++j) bf[j] = B[tr][32 * wn + 8 * j + (lane >> 2)];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
    __syncthreads();
  }
  double* out = W + ((size_t)blockIdx.y * gridDim.x + blockIdx.x) * 4096;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int row = 32 * wm + 8 * i + (lane >> 2);
      const int col = 32 * wn + 8 * j + 2 * (lane & 3);
      *reinterpret_cast<double2*>(out + row * 64 + col) = make_double2(acc[i][j][0], acc[i][j][1]);
    }
  __shared__ int s_last;
  __threadfence();
  __syncthreads();
  if (tid == 0) {
    const int prev = atomicAdd(tickets + blockIdx.x, 1);
    s_last = prev == (int)gridDim.y - 1;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  const int nsplit = gridDim.y;
  // valid elements only; partials summed in split order, 8 elements in flight per thread
  const double* wp = W + (size_t)blockIdx.x * 4096;
  const size_t sstride = (size_t)gridDim.x * 4096;
  const int nr = min(64, K - J0), nc = min(64, K - L0);
  const int nvalid = nr * nc;
  for (int e0 = tid; e0 < nvalid; e0 += 8 * kGramThreads) {
    double s[8];
    int el[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = e0 + u * kGramThreads;
      s[u] = 0.0;
      el[u] = e < nvalid ? (e / nc) * 64 + (e % nc) : -1;
    }
    for (int sp = 0; sp < nsplit; ++sp) {
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (el[u] >= 0) s[u] += __ldcg(wp + sp * sstride + el[u]);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (el[u] >= 0) {
        const int row = J0 + (el[u] >> 6), col = L0 + (el[u] & 63);
        if (row <= col || (row >> 5) == (col >> 5)) G[tpu_idx(K, row, col)] = s[u];  // TPU output
      }
  }
  if (tid == 0) tickets[blockIdx.x] = 0;
}

constexpr int kQA = 36;

// Q[t][l] = sum_{a <= l} A(t, a) * B(a, l), l < K, for an upper-triangular
// TPU right factor B (CholeskyQR's Q = A R^-1, or A T with the carried
// preconditioner).
template <class L>
__global__ void __launch_bounds__(kGramThreads)
    k_qform(L ld, int64_t rows, int K, const double* __restrict__ B, double* __restrict__ Q,
            int64_t ldq, const int* skip_flag) {
  if (skip_flag && *skip_flag == 0) return;
  __shared__ __align__(16) double SA[64][kQA];
  __shared__ __align__(16) double SR[32][kSJ];
  const int64_t t0 = (int64_t)blockIdx.x * 64;
  const int L0 = blockIdx.y * 64;
  const int jend = min(K, L0 + 64);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp & 1, wn = warp >> 1;
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  for (int k0 = 0; k0 < jend; k0 += 32) {
    {
      const int cc = tid & 31, rr0 = tid >> 5;
#pragma unroll 4
      for (int s = 0; s < 16; ++s) {
        const int rr = rr0 + 4 * s;
        const int64_t row = t0 + rr;
        SA[rr][cc] = (row < rows && k0 + cc < K) ? ld(row, k0 + cc) : 0.0;
      }
      const int ll = tid & 63, c0 = tid >> 6;
#pragma unroll 4
      for (int s = 0; s < 16; ++s) {
        const int c = c0 + 2 * s;
        const int r = k0 + c, cl = L0 + ll;
        SR[c][ll] = (r < K && cl < K && r <= cl) ? B[tpu_idx(K, r, cl)] : 0.0;
      }
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      double af[4], bf[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) af[i] = SA[32 * wm + 8 * i + (lane >> 2)][4 * kk + (lane & 3)];
#pragma unroll
      for (int j = 0; j < 4; ++j) bf[j] = SR[4 * kk + (lane & 3)][32 * wn + 8 * j + (lane >> 2)];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t row = t0 + 32 * wm + 8 * i + (lane >> 2);
      const int col = L0 + 32 * wn + 8 * j + 2 * (lane & 3);
      if (row < rows) {
        if (col < K) Q[row * ldq + col] = acc[i][j][0];
        if (col + 1 < K) Q[row * ldq + col + 1] = acc[i][j][1];
      }
    }
}

}  // namespace tfk
