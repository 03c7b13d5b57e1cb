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
// Transform of a batch of columns, in passes of up to 8 levels (strides
// 2^l0 .. 2^(l1-1)) through shared memory: a CTA holds the 2^(l1-l0)
// elements of one butterfly group for LW = min(16, 2^l0) consecutive
// low offsets (128-byte coalesced rows), i = lo + mid 2^l0 + hi 2^l1.  The
// first pass builds sign(i) * y[i + a] on load (column a of the forward
// column order is y[i + a]; a = h is the target).
#pragma once

#include "common.cuh"

namespace tfk {

constexpr int kFwhtThreads = 256;
constexpr int kFwhtMaxLevels = 8;   // strided passes
constexpr int kFwhtMaxFirst = 11;   // contiguous pass (l0 = 0)

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

__global__ void __launch_bounds__(kFwhtThreads) k_fwht_pass(FwhtArgs a) {
  extern __shared__ double T[];  // [M][LW]
  const int L = a.l1 - a.l0;
  const int M = 1 << L;
  const int LW = a.l0 >= 4 ? 16 : (1 << a.l0);
  const int64_t nlo = ((int64_t)1 << a.l0) / LW;  // low-offset groups
  const int64_t tile = blockIdx.x;
  const int64_t lo_base = (tile % nlo) * LW;
  const int64_t hi = tile / nlo;
  double* X = a.X + (int64_t)blockIdx.y * a.N;
  const int n = M * LW;
  auto gidx = [&](int e) { return lo_base + (e % LW) + ((int64_t)(e / LW) << a.l0) + (hi << a.l1); };
  if (a.y) {
    const double* src = a.y + a.a0 + blockIdx.y;
    for (int e = threadIdx.x; e < n; e += kFwhtThreads) {
      const int64_t i = gidx(e);
      double v = 0.0;
      if (i < a.n0) v = (rng_draw(a.seed, (uint64_t)i) >> 63) ? src[i] : -src[i];
      T[e] = v;
    }
  } else {
    for (int e = threadIdx.x; e < n; e += kFwhtThreads) T[e] = X[gidx(e)];
  }
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
  for (int e = threadIdx.x; e < n; e += kFwhtThreads) X[gidx(e)] = T[e];
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
