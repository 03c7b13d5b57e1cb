// k_srht.cuh -- subsampled randomized Hadamard transform path (SURVEY 8(f)
// item 4; sketch.cpp:103-239, bench.cpp:50-72).
//
// Per lag h the reference signs the n0 = n - h rows of [X_h | y] with the
// first n0 draws of Rng(derive_seed(seed, h)), zero-pads to N = bit_ceil(n0),
// applies the orthonormal Walsh-Hadamard transform (butterflies
// (a + b) / sqrt(2), (a - b) / sqrt(2)) and keeps the rows below(N) drawn
// next, weighted sqrt(N / c).  Its pruned transform (PartialHadamard) runs
// the levels from the LARGEST stride down; the passes here do the same, so
// the sampled rows are bit-identical to the reference's.
//
// Transform of a batch of columns, in passes of 8 levels from the top
// (strides 2^l0 .. 2^(l0+7)) through shared memory: a CTA holds the 256
// elements of a butterfly group for 16 lanes (16 consecutive low offsets:
// 128-byte coalesced rows, i = lo + mid 2^l0 + hi 2^(l0+8); for l0 = 0,
// 16 consecutive 256-element groups), and runs the 8 levels as two rounds of
// 4 in registers (16 elements per thread).  The last pass takes the
// remaining < 8 levels.  The first pass builds sign(i) * y[i + a] on load
// (column a of the forward column order is y[i + a]; a = h is the target).
#pragma once

#include "common.cuh"

namespace tfk {

constexpr int kFwhtThreads = 256;
constexpr int kFwhtLevels = 8;  // levels per pass (the last pass takes the remainder)

// c draws of below(N) that follow the n0 sign draws; N a power of two, so
// below() rejects x >= 2^64 - N (probability N / 2^64): flagged, host redraws
__global__ void k_srht_draws(uint64_t seed, int64_t n0, int64_t N, int64_t c, int64_t* __restrict__ draws,
                             int* reject) {
  const uint64_t limit = 0ull - (uint64_t)N;  // 2^64 - N
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < c; t += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t x = rng_draw(seed, (uint64_t)(n0 + t));
    if (x >= limit) atomicExch(reject, 1);
    draws[t] = (int64_t)(x & (uint64_t)(N - 1));
  }
}

struct FwhtArgs {
  double* X;          // batch: column b at X + b * N
  int64_t N;
  int l0, l1;         // levels [l0, l1) of this pass
  // first pass only (y != nullptr): x_b[i] = sign(i) * y[i + a0 + b] for i < n0
  const double* y;
  int64_t n0;
  int a0;
  uint64_t seed;
};

// Fast pass: 8 levels, 16 lanes (low offsets, or for l0 = 0 sixteen
// consecutive groups), tile T[mid][16] of 4096 doubles; the 8 levels run as
// two register rounds of 4 (mid bits 7..4, then 3..0: largest stride first),
// each thread holding 16 elements of one lane.
__device__ __forceinline__ void fwht_reg16(double (&v)[16]) {
  const double s = 0.70710678118654752440;
#pragma unroll
  for (int b = 3; b >= 0; --b) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      if (k & (1 << b)) continue;
      const double x0 = v[k], x1 = v[k | (1 << b)];
      v[k] = (x0 + x1) * s;
      v[k | (1 << b)] = (x0 - x1) * s;
    }
  }
}

__global__ void __launch_bounds__(kFwhtThreads) k_fwht_pass(FwhtArgs a) {
  extern __shared__ double T[];  // [M][LW]
  const int L = a.l1 - a.l0;
  double* X = a.X + (int64_t)blockIdx.y * a.N;
  const double* src = a.y ? a.y + a.a0 + blockIdx.y : nullptr;
  auto load = [&](int64_t i) -> double {
    if (!src) return X[i];
    if (i >= a.n0) return 0.0;
    return (rng_draw(a.seed, (uint64_t)i) >> 63) ? src[i] : -src[i];
  };
  if (L == 8 && (a.l0 == 0 || a.l0 >= 4) && a.N >= 4096) {
    // element (lane, mid): l0 >= 4: i = lo_base + lane + mid 2^l0 + hi 2^(l0 + 8)
    //                      l0 = 0:  i = mid + (hi_base + lane) 2^8
    int64_t base;
    int64_t lstride, mstride;
    if (a.l0 == 0) {
      base = (int64_t)blockIdx.x * 4096;
      lstride = 256;
      mstride = 1;
    } else {
      const int64_t nlo = ((int64_t)1 << a.l0) / 16;
      base = (blockIdx.x % nlo) * 16 + ((int64_t)(blockIdx.x / nlo) << (a.l0 + 8));
      lstride = 1;
      mstride = (int64_t)1 << a.l0;
    }
    for (int e = threadIdx.x; e < 4096; e += kFwhtThreads) {
      const int lane = e & 15, mid = e >> 4;
      T[e] = load(base + lane * lstride + mid * mstride);
    }
    __syncthreads();
    const int lane = threadIdx.x & 15, g = threadIdx.x >> 4;
    double v[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) v[k] = T[(g + 16 * k) * 16 + lane];  // mid bits 7..4 vary
    fwht_reg16(v);
#pragma unroll
    for (int k = 0; k < 16; ++k) T[(g + 16 * k) * 16 + lane] = v[k];
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 16; ++k) v[k] = T[(16 * g + k) * 16 + lane];  // mid bits 3..0 vary
    fwht_reg16(v);
#pragma unroll
    for (int k = 0; k < 16; ++k) T[(16 * g + k) * 16 + lane] = v[k];
    __syncthreads();
    for (int e = threadIdx.x; e < 4096; e += kFwhtThreads) {
      const int ln = e & 15, mid = e >> 4;
      X[base + ln * lstride + mid * mstride] = T[e];
    }
    return;
  }
  // generic pass (fewer than 8 levels): lanes are low offsets (l0 > 0) or,
  // for l0 = 0, consecutive groups of 2^L contiguous elements
  const int M = 1 << L;
  int LW;
  int64_t base, lstride, mstride;
  if (a.l0 == 0) {
    LW = (int)min((int64_t)max(1, 4096 / M), a.N / M);
    base = (int64_t)blockIdx.x * LW * M;
    lstride = M;
    mstride = 1;
  } else {
    LW = a.l0 >= 4 ? 16 : (1 << a.l0);
    const int64_t nlo = ((int64_t)1 << a.l0) / LW;
    base = (blockIdx.x % nlo) * LW + ((int64_t)(blockIdx.x / nlo) << a.l1);
    lstride = 1;
    mstride = (int64_t)1 << a.l0;
  }
  const int n = M * LW;
  for (int e = threadIdx.x; e < n; e += kFwhtThreads) T[e] = load(base + (e % LW) * lstride + (e / LW) * mstride);
  __syncthreads();
  const double s = 0.70710678118654752440;
  for (int k = L - 1; k >= 0; --k) {  // largest stride first
    const int bit = 1 << k;
    for (int p = threadIdx.x; p < n / 2; p += kFwhtThreads) {
      const int lo = p % LW, q = p / LW;
      const int mid = ((q >> k) << (k + 1)) | (q & (bit - 1));
      const int e0 = mid * LW + lo, e1 = (mid | bit) * LW + lo;
      const double x0 = T[e0], x1 = T[e1];
      T[e0] = (x0 + x1) * s;
      T[e1] = (x0 - x1) * s;
    }
    __syncthreads();
  }
  for (int e = threadIdx.x; e < n; e += kFwhtThreads) X[base + (e % LW) * lstride + (e / LW) * mstride] = T[e];
}

// D[t][a0 + b] = w * X_b[draws[t]] (row-major, ld)
__global__ void k_srht_gather(const double* __restrict__ X, int64_t N, int nb, const int64_t* __restrict__ draws,
                              int64_t c, double w, double* __restrict__ D, int64_t ld, int a0) {
  const int64_t tot = c * nb;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = e / nb;
    const int b = (int)(e % nb);
    D[t * ld + a0 + b] = w * X[(int64_t)b * N + draws[t]];
  }
}

}  // namespace tfk
