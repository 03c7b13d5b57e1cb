// common.cuh -- device helpers shared by the toepfit B200 kernels.
//
// * Counter RNG bit-identical to the reference's Rng (rng.hpp:14-84): draw t
//   (0-based) of Rng(s) is mix(s + (t+1) * golden), so any draw is computable
//   independently on any thread.
// * DMMA (mma.sync m8n8k4 f64) wrapper -- the fp64 tensor-core instruction on
//   sm_100a (SASS: DMMA.8x8x4).  Fragment layout (PTX ISA, m8n8k4 .f64):
//     A (8x4, row):  a = A[lane>>2][lane&3]
//     B (4x8, col):  b = B[lane&3][lane>>2]
//     C (8x8):       c0,c1 = C[lane>>2][2*(lane&3) + {0,1}]
// * Warp inclusive scans / reductions in a fixed order (deterministic).
#pragma once

#include <type_traits>

#include <cstdint>
#include <cuda_runtime.h>

namespace tfk {

constexpr uint64_t kGolden = 0x9e3779b97f4a7c15ull;

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

// derive_seed(seed, tag) = Rng(seed).fork(tag)()  (rng.hpp:30-32, 82-84)
__host__ __device__ __forceinline__ uint64_t derive_seed(uint64_t seed, uint64_t tag) {
  const uint64_t child = mix64(seed ^ mix64(tag + 0x632be59bd9b4e019ull));
  return mix64(child + kGolden);
}

// raw draw t (0-based) of Rng(seed)
__host__ __device__ __forceinline__ uint64_t rng_draw(uint64_t seed, uint64_t t) {
  return mix64(seed + (t + 1) * kGolden);
}

// uniform01 of draw t (rng.hpp:35): 53 random bits
__host__ __device__ __forceinline__ double rng_uniform01(uint64_t seed, uint64_t t) {
  return static_cast<double>(rng_draw(seed, t) >> 11) * 0x1.0p-53;
}

__device__ __forceinline__ void dmma_8x8x4(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// 4 x 4 DMMA block acc[i][j] += a[i] b[j].  FULL: every product (no
// predicates).  Otherwise only i < ni, j < nj; a predicated mma.sync costs a
// WARPSYNC + NOP + compare per DMMA, so callers branch to FULL (warp-uniformly)
// whenever the whole block is live.
template <bool FULL>
__device__ __forceinline__ void dmma_4x4(double (&acc)[4][4][2], const double (&a)[4], const double (&b)[4], int ni,
                                         int nj) {
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (FULL || (i < ni && j < nj)) dmma_8x8x4(acc[i][j][0], acc[i][j][1], a[i], b[j]);
}

// Division-free reciprocal / reciprocal square root: MUFU approximation plus
// two Newton steps (error ~1 ulp).  Used inside fully unrolled register code
// where the IEEE division slow-path call would force arrays into local memory.
__device__ __forceinline__ double fast_rcp(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}

__device__ __forceinline__ double fast_rsqrt(double x) {
  double r;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  const double hx = 0.5 * x;
  double t = fma(-hx * r, r, 0.5);
  r = fma(r, t, r);
  t = fma(-hx * r, r, 0.5);
  return fma(r, t, r);
}

// ---- bulk async copies (cp.async.bulk, TMA engine) with an mbarrier ----
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  uint32_t done = 0;
  do {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(phase)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
               "r"(smem_u32(src)), "r"(bytes)
               : "memory");
}
// DRAM -> L2 bulk prefetch (no shared memory, no registers); bytes % 16 == 0
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_commit_wait_all() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// inclusive scan across lanes (Kogge-Stone, fixed order)
__device__ __forceinline__ double warp_incl_scan(double v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double u = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += u;
  }
  return v;
}

}  // namespace tfk
