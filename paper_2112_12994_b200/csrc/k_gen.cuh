// k_gen.cuh -- on-device synthetic AR series: the
// BASELINE root-based cascade generator, x_t = x_{t-1} / r_k + in_t for each
// real root r_k, run as parallel linear-recurrence scans so that n = 1e9
// series (C4) never cross PCIe.  Innovations from the reference's counter RNG
// (rng.hpp:23-35 draws): Box-Muller normals, or Student-t(3) / sqrt(3).
//
// Scan of x_t = a x_{t-1} + u_t (|a| < 1): each thread folds 8 consecutive
// elements, the CTA combines its threads' (a^8, carry) pairs with an affine
// warp/block scan, a single-CTA pass propagates block carries, and a final
// pass adds a^(t - t_block + 1) * carry_in to every element.  Rounding differs
// from a sequential filter (a generator, not a parity object).
#pragma once

#include "common.cuh"

namespace tfk {

constexpr int kGenThreads = 256;
constexpr int kGenPer = 8;
constexpr int kGenBlock = kGenThreads * kGenPer;  // 2048 elements per CTA

__global__ void k_gen_innovations(uint64_t seed, int64_t total, int t3, double* __restrict__ out) {
  const double two_pi = 6.283185307179586476925286766559;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; 2 * j < total;
       j += (int64_t)gridDim.x * blockDim.x) {
    if (!t3) {
      const double u1 = rng_uniform01(seed, 2 * (uint64_t)j) + 0x1.0p-54;  // (0, 1]
      const double u2 = rng_uniform01(seed, 2 * (uint64_t)j + 1);
      const double rad = sqrt(-2.0 * log(u1));
      double sn, cs;
      sincos(two_pi * u2, &sn, &cs);
      out[2 * j] = rad * cs;
      if (2 * j + 1 < total) out[2 * j + 1] = rad * sn;
    } else {
      // two t3 / sqrt(3) values per pair: each from 4 normals (z / sqrt(chi2_3 / 3) / sqrt(3))
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        if (2 * j + h >= total) break;
        double z[4];
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const uint64_t base = 8 * (uint64_t)j + 4 * h + 2 * q;
          const double u1 = rng_uniform01(seed, base) + 0x1.0p-54;
          const double u2 = rng_uniform01(seed, base + 1);
          const double rad = sqrt(-2.0 * log(u1));
          double sn, cs;
          sincos(two_pi * u2, &sn, &cs);
          z[2 * q] = rad * cs;
          z[2 * q + 1] = rad * sn;
        }
        const double chi = z[1] * z[1] + z[2] * z[2] + z[3] * z[3];
        out[2 * j + h] = z[0] / sqrt(chi / 3.0) / sqrt(3.0);
      }
    }
  }
}

// phase 1: in-CTA scan of x_t = a x_{t-1} + x_t (zero carry in); block end value -> bend
__global__ void __launch_bounds__(kGenThreads) k_ar_scan_local(double* __restrict__ x, int64_t n, double a,
                                                               double* __restrict__ bend) {
  __shared__ double sv[kGenThreads];
  const int tid = threadIdx.x;
  const int64_t base = (int64_t)blockIdx.x * kGenBlock + (int64_t)tid * kGenPer;
  double v[kGenPer];
  double c = 0.0;
#pragma unroll
  for (int u = 0; u < kGenPer; ++u) {
    const double in = base + u < n ? x[base + u] : 0.0;
    c = fma(a, c, in);
    v[u] = c;
  }
  // thread prefix: carry_t = a^8 carry_{t-1} + c_t  (Hillis-Steele with powers)
  double a8 = a;
#pragma unroll
  for (int u = 1; u < kGenPer; ++u) a8 *= a;  // a^8
  sv[tid] = c;
  __syncthreads();
  double mult = a8;  // a^(8 * offset)
  for (int off = 1; off < kGenThreads; off <<= 1) {
    const double prev = tid >= off ? sv[tid - off] : 0.0;
    __syncthreads();
    if (tid >= off) sv[tid] = fma(mult, prev, sv[tid]);
    __syncthreads();
    mult *= mult;
  }
  const double cin = tid > 0 ? sv[tid - 1] : 0.0;  // carry into this thread's segment
  double ap = a;
#pragma unroll
  for (int u = 0; u < kGenPer; ++u) {
    if (base + u < n) x[base + u] = fma(ap, cin, v[u]);
    ap *= a;
  }
  if (tid == kGenThreads - 1) bend[blockIdx.x] = sv[tid];
}

// phase 2: single CTA, carries across blocks: cin_b = a^B cin_{b-1} + bend_{b-1}
__global__ void __launch_bounds__(1024) k_ar_scan_blocks(double* __restrict__ bend, int64_t nblk, double aB) {
  __shared__ double seg_end[1024], seg_mul[1024];
  const int tid = threadIdx.x;
  const int64_t per = (nblk + 1023) / 1024;
  const int64_t b0 = min(nblk, (int64_t)tid * per), b1 = min(nblk, b0 + per);
  double c = 0.0, m = 1.0;  // local fold of this thread's blocks (zero carry in)
  for (int64_t b = b0; b < b1; ++b) {
    c = fma(aB, c, bend[b]);
    m *= aB;
  }
  seg_end[tid] = c;
  seg_mul[tid] = m;
  __syncthreads();
  if (tid == 0) {  // sequential over the 1024 segment summaries
    double carry = 0.0;
    for (int t = 0; t < 1024; ++t) {
      const double e = seg_end[t], mm = seg_mul[t];
      seg_end[t] = carry;  // carry into segment t
      carry = fma(mm, carry, e);
    }
  }
  __syncthreads();
  double carry = seg_end[tid];
  for (int64_t b = b0; b < b1; ++b) {
    const double e = bend[b];
    bend[b] = carry;  // carry into block b
    carry = fma(aB, carry, e);
  }
}

// phase 3: x_t += a^(t - t_b + 1) cin_b
__global__ void __launch_bounds__(kGenThreads) k_ar_scan_apply(double* __restrict__ x, int64_t n, double a,
                                                               const double* __restrict__ cin) {
  const double c = cin[blockIdx.x];
  if (c == 0.0) return;
  const int tid = threadIdx.x;
  const int64_t base = (int64_t)blockIdx.x * kGenBlock + (int64_t)tid * kGenPer;
  // a^(8 tid + 1) by binary exponentiation
  double ap = 1.0, bsq = a;
  for (int e = kGenPer * tid + 1; e > 0; e >>= 1) {
    if (e & 1) ap *= bsq;
    bsq *= bsq;
  }
#pragma unroll
  for (int u = 0; u < kGenPer; ++u) {
    if (base + u < n) x[base + u] = fma(ap, c, x[base + u]);
    ap *= a;
  }
}

}  // namespace tfk
