// k_i8gram.cuh -- the double-double Gram of the sampled rows on the INT8
// tensor cores (tcgen05.mma kind::i8, TMEM accumulators): an exact-product
// (Ozaki-style) splitting.
//
// Column j of A (the gathered, weighted rows) is scaled by 2^-E_j (E_j from the
// column's max |a|, so |x| < 1/2) and written as S signed 7-bit digits,
//   a_tj = 2^E_j sum_{s<S} d_s,tj 2^{-7 (s+1)},  d in [-64, 64]
// (exact for every entry within 2^{7S-53} of the column max; the truncation of
// smaller entries is below 2^{E_j - 7S - 1}).  The digit planes are stacked as
// columns of one int8 matrix D (S Kp columns, K-major: each column's rows
// contiguous), and
//   G_ij = sum_{s,u} 2^{E_i + E_j - 7 (s + u + 2)} P[(s, i), (u, j)],  P = D^T D
// with P exact in int32 (|d d'| <= 2^12, c <= 2^19 rows).  Only the blocks with
// s + u <= S - 1 are formed (the rest lie below the truncation); the powers of
// two and the sum run in double-double (k_i8_combine), so G comes out as the
// same (hi, lo) pair k_gram_dd produces -- to ~1e-26 relative with S = 14.
//
// GEMM: one CTA (128 threads) per 128 x 128 output tile of P, tile pairs
// (I <= J) from a host list; 128-row (128-byte) K steps staged by cp.async into
// a 4-stage shared-memory ring in the UMMA K-major "interleave" layout (8-row x
// 16-byte core matrices); one elected thread issues 4 tcgen05.mma (M = N = 128,
// K = 32) per step and commits them to the stage's mbarrier (the ring slot is
// refilled once the MMAs reading it completed); the int32 accumulator lives in
// TMEM (128 columns) and is read back with tcgen05.ld for the epilogue.
#pragma once

#include <cstdint>

#include "common.cuh"
#include "k_exact.cuh"

namespace tfk {

constexpr int kI8S = 14;          // digit planes (98 bits)
constexpr int kI8Tile = 128;      // output tile (stacked columns) and K step (rows)
constexpr int kI8Stages = 4;
constexpr int kI8Threads = 128;
constexpr int kI8N = 256;                         // output tile: 128 stacked columns (I) x 256 (J pair)
constexpr size_t kI8StageBytes = 3 * 128 * 128;  // A block + two B blocks per stage
constexpr size_t kI8Smem = kI8Stages * kI8StageBytes + 1024;
constexpr int64_t kI8MaxRows = 1LL << 19;  // |sum of c digit products| <= 2^12 c < 2^31
constexpr double kI8MinWork = 4e8;         // c K^2 above which the tensor-core Gram is faster (B200)
constexpr int kI8Bad = 1 << 20;            // E_j of a column holding a NaN / Inf

__device__ __forceinline__ double fmax_nan(double a, double b) { return (b > a || b != b) ? b : a; }  // NaN sticks

__device__ __forceinline__ uint32_t i8_smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// column max |a| (partials per row block) -> exponent E_j with max |a| * 2^-E_j < 1/2
template <class L>
__global__ void __launch_bounds__(256) k_i8_colmax_part(L ld, int64_t rows, int K, const long long* rows_dev,
                                                        double* __restrict__ part) {
  if (rows_dev) rows = min(rows, (int64_t)*rows_dev);
  __shared__ double red[4][64];
  const int tid = threadIdx.x, col = 64 * blockIdx.x + (tid & 63), rg = tid >> 6;
  const int64_t r0 = (int64_t)blockIdx.y * kCnRows, r1 = min(rows, r0 + kCnRows);
  double m = 0.0;
  if (col < K)
    for (int64_t t = r0 + rg; t < r1; t += 4) {
      const double a = fabs(ld(t, col));
      m = (a > m || a != a) ? a : m;  // NaN sticks
    }
  red[rg][tid & 63] = m;
  __syncthreads();
  if (tid < 64 && col < K) {
    double v = red[0][tid];
    for (int g = 1; g < 4; ++g) v = (red[g][tid] > v || red[g][tid] != red[g][tid]) ? red[g][tid] : v;
    part[(int64_t)blockIdx.y * K + col] = v;
  }
}
__global__ void k_i8_colmax_fin(const double* __restrict__ part, int nsplit, int K, int* __restrict__ E) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= K) return;
  double m = 0.0;
  for (int sp = 0; sp < nsplit; ++sp) {
    const double v = part[(int64_t)sp * K + j];
    m = (v > m || v != v) ? v : m;
  }
  if (!isfinite(m)) {
    E[j] = kI8Bad;  // k_i8_combine writes NaN into the column (as the double-double Gram would)
    return;
  }
  int e = 0;
  if (m > 0.0) frexp(m, &e);  // m < 2^e
  E[j] = e + 1;               // |a| 2^-E < 1/2
}

// Window-system rows (FwdRows: a_tj = w_t y[idx_t + j]): one exponent for
// every column from the bound max_t |w_t| * max_i |y_i| (no pass over the c x K
// sampled entries).  The bound exceeds a column's own max by a few bits at
// most (same series, same weights), which the 98-bit digit budget absorbs.
// ybits: max |y| as the bit pattern of a non-negative double (k_absmax_bits).
__global__ void k_absmax_bits(const double* __restrict__ y, int64_t n, unsigned long long* __restrict__ out) {
  double m = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double a = fabs(__ldg(y + i));
    m = (a > m || a != a) ? a : m;
  }
  m = fmax_nan(m, __shfl_xor_sync(0xffffffffu, m, 16));
  m = fmax_nan(m, __shfl_xor_sync(0xffffffffu, m, 8));
  m = fmax_nan(m, __shfl_xor_sync(0xffffffffu, m, 4));
  m = fmax_nan(m, __shfl_xor_sync(0xffffffffu, m, 2));
  m = fmax_nan(m, __shfl_xor_sync(0xffffffffu, m, 1));
  if ((threadIdx.x & 31) == 0) atomicMax(out, (unsigned long long)__double_as_longlong(m));  // order-free
}
__global__ void __launch_bounds__(1024) k_i8_exp_fwd(const double* __restrict__ wt, int64_t rows,
                                                     const long long* rows_dev,
                                                     const unsigned long long* __restrict__ ybits, int K,
                                                     int* __restrict__ E) {
  if (rows_dev) rows = min(rows, (int64_t)*rows_dev);
  __shared__ double red[32];
  double m = 0.0;
  for (int64_t t = threadIdx.x; t < rows; t += blockDim.x) {
    const double a = fabs(wt[t]);
    m = (a > m || a != a) ? a : m;
  }
  for (int o = 16; o > 0; o >>= 1) m = fmax_nan(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x < 32) {
    m = red[threadIdx.x];
    for (int o = 16; o > 0; o >>= 1) m = fmax_nan(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (threadIdx.x == 0) red[0] = m;
  }
  __syncthreads();
  const double bound = red[0] * __longlong_as_double((long long)*ybits) * (1.0 + 0x1p-40);
  int e = 0;
  if (bound > 0.0 && isfinite(bound)) frexp(bound, &e);
  const int ev = isfinite(bound) ? e + 1 : kI8Bad;
  for (int j = threadIdx.x; j < K; j += blockDim.x) E[j] = ev;
}

__device__ __forceinline__ uint64_t i8_sdesc(uint32_t addr) {
  // K-major, no swizzle: LBO = 128 B (next 16-byte K chunk), SBO = 1024 B (next 8-row group)
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)(128 >> 4) << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;  // descriptor version (sm_100)
  return d;
}

// byte offset of (row r of a block = stacked column, byte kb of the 128-row K step)
__host__ __device__ __forceinline__ int i8_lay(int r, int kb) {
  return (r >> 3) * 1024 + (kb >> 4) * 128 + (r & 7) * 16 + (kb & 15);
}

// digit planes, pre-tiled: block (Ib, k) of 128 stacked columns x 128 rows is
// 16 KB at D + (Ib nk + k) 16384 in the UMMA K-major interleave layout
// (i8_lay), so one bulk copy stages it; stacked column Ib 128 + r = s Kp + j.
// Rows past `rows` and columns past K are zero.  One CTA: 32 columns x 128 rows.
template <class L>
__global__ void __launch_bounds__(256) k_i8_slice(L ld, int64_t rows, int K, int Kp, int64_t nk,
                                                  const long long* rows_dev, const int* __restrict__ E,
                                                  int8_t* __restrict__ D) {
  if (rows_dev) rows = min(rows, (int64_t)*rows_dev);
  const int j = blockIdx.y * 32 + (threadIdx.x & 31);
  const int64_t k = blockIdx.x;
  const int kb0 = (threadIdx.x >> 5) * 16;
  const int64_t t0 = k * kI8Tile + kb0;
  int ej = j < K ? E[j] : 0;
  if (ej == kI8Bad) ej = 0;  // digits are don't-cares: the column's Gram entries become NaN
  // 2^-E as a multiplier (exact; ldexp only outside the normal exponent range)
  const bool plain = ej > -1022 && ej < 1022;
  const double sc = __longlong_as_double((long long)(1023 - ej) << 52);
  double x[16];
#pragma unroll
  for (int u = 0; u < 16; ++u) {
    const int64_t t = t0 + u;
    double a = 0.0;
    if (j < K && t < rows) {
      const double v = ld(t, j);
      a = plain ? v * sc : ldexp(v, -ej);
    }
    x[u] = isfinite(a) && fabs(a) < 0.5 ? a : 0.0;
  }
  const int nbs = Kp / kI8Tile;
  // d = round-half-even(y) by the 1.5 * 2^52 shifter: y + M holds d in its low
  // mantissa bits (|y| <= 64) and (y + M) - M = d exactly -- the digits rint /
  // cvt give, in fp64 adds only
  constexpr double kShift = 6755399441055744.0;  // 1.5 * 2^52
#pragma unroll 1
  for (int s = 0; s < kI8S; ++s) {
    uint32_t w[4] = {0u, 0u, 0u, 0u};
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      // 128 x is exact (power of two), so the two fused operations round exactly what the
      // separate multiply + add / subtract did -- the same digits in 3 fp64 operations instead of 4
      // (the kernel is bound by the fp64 pipe)
      const double m = __fma_rn(x[u], 128.0, kShift);
      const double d = __dsub_rn(m, kShift);
      x[u] = __fma_rn(x[u], 128.0, -d);  // exact: 128 x and d share the exponent range
      w[u >> 2] |= ((uint32_t)__double2loint(m) & 0xFFu) << (8 * (u & 3));
    }
    const int64_t Ib = (int64_t)s * nbs + j / kI8Tile;
    *reinterpret_cast<uint4*>(D + (Ib * nk + k) * 16384 + i8_lay(j % kI8Tile, kb0)) = make_uint4(w[0], w[1], w[2], w[3]);
  }
}

__device__ __forceinline__ void i8_mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t done = 0;
  while (!done)
    asm volatile("{\n\t.reg .pred P;\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n\tselp.b32 %0, 1, 0, P;\n\t}"
                 : "=r"(done) : "r"(bar), "r"(parity) : "memory");
}

// P tiles: out[tile][128][256] int32 (row = stacked column of block I, col =
// stacked column of blocks 2m, 2m + 1).  One CTA per tile (I, m): per 128-row
// K step three 16 KB bulk copies (block I, blocks 2m and 2m + 1, which land
// contiguously = one 256-row K-major B operand) into a kI8Stages ring; warp 0
// lane 0 streams (full barrier: transaction bytes; empty barrier: the MMAs'
// commit), warp 1 lane 0 issues 4 tcgen05.mma (M = 128, N = 256, K = 32) per
// step; all four warps drain the 256 TMEM columns.  N = 256 halves the operand
// bytes per MMA of the 128 x 128 version (the kernel was feeding its tensor
// pipe at 37 % from L2 at 14.8 TB/s; profiles/r02_i8_gemm.txt).
// Split K (few tiles, small K): CTA blockIdx.x covers tile blockIdx.x % ntiles
// over the K steps of split blockIdx.x / ntiles and writes its partial tile to
// out[split][tile]; k_i8_combine adds the splits (int32: every partial is
// bounded like the whole sum).
__global__ void __launch_bounds__(kI8Threads) k_i8_gemm(const int8_t* __restrict__ D, int64_t nk,
                                                        const int2* __restrict__ tiles, int32_t* __restrict__ out,
                                                        int ntiles, int ksplit) {
  extern __shared__ __align__(1024) unsigned char i8sm[];
  __shared__ __align__(8) uint64_t full[kI8Stages], empty[kI8Stages], done;
  __shared__ uint32_t tmem_base;
  unsigned char* base = i8sm + ((1024 - (i8_smem_u32(i8sm) & 1023)) & 1023);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int tile = (int)(blockIdx.x % (unsigned)ntiles), split = (int)(blockIdx.x / (unsigned)ntiles);
  const int2 tp = tiles[tile];  // (I, m)
  const int64_t kb = nk * split / ksplit, ke = nk * (split + 1) / ksplit;  // this CTA's K steps [kb, ke)
  const int8_t* blkA = D + (int64_t)tp.x * nk * 16384;
  const int8_t* blkB0 = D + (int64_t)(2 * tp.y) * nk * 16384;
  const int8_t* blkB1 = D + (int64_t)(2 * tp.y + 1) * nk * 16384;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(i8_smem_u32(&tmem_base)),
                 "r"(kI8N));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 32) {
    for (int s = 0; s < kI8Stages; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(i8_smem_u32(&full[s])), "r"(1));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(i8_smem_u32(&empty[s])), "r"(1));
    }
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(i8_smem_u32(&done)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base;
  if (tid == 0) {  // producer
    for (int64_t k = 0; k < ke - kb; ++k) {
      const int st = (int)(k % kI8Stages);
      if (k >= kI8Stages) i8_mbar_wait(i8_smem_u32(&empty[st]), (uint32_t)(((k / kI8Stages) - 1) & 1));
      const uint32_t fb = i8_smem_u32(&full[st]);
      const uint32_t sA = i8_smem_u32(base + (size_t)st * kI8StageBytes);
      const int64_t kg = kb + k;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(fb), "r"(3u * 16384u) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sA),
                   "l"(blkA + kg * 16384), "r"(16384), "r"(fb) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       sA + 16384), "l"(blkB0 + kg * 16384), "r"(16384), "r"(fb) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       sA + 32768), "l"(blkB1 + kg * 16384), "r"(16384), "r"(fb) : "memory");
    }
  } else if (tid == 32) {  // MMA issuer
    // instruction descriptor: D s32, A / B s8, K-major, N = 256 (n_dim 32), M = 128 (m_dim 8)
    const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(kI8N >> 3) << 17) | (8u << 24);
    for (int64_t k = 0; k < ke - kb; ++k) {
      const int st = (int)(k % kI8Stages);
      i8_mbar_wait(i8_smem_u32(&full[st]), (uint32_t)((k / kI8Stages) & 1));
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t a0 = i8_smem_u32(base + (size_t)st * kI8StageBytes), b0 = a0 + 16384;
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {  // K = 32 bytes per MMA: 2 chunks of 16
        const uint64_t da = i8_sdesc(a0 + kk * 256), db = i8_sdesc(b0 + kk * 256);
        const uint32_t acc = (k > 0 || kk > 0) ? 1u : 0u;
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
                     "l"(da), "l"(db), "r"(idesc), "r"(acc));
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          i8_smem_u32(&empty[st])));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(i8_smem_u32(&done)));
  }
  __syncwarp();
  i8_mbar_wait(i8_smem_u32(&done), 0u);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  int32_t* o = out + (size_t)blockIdx.x * 128 * kI8N + (size_t)(32 * warp + lane) * kI8N;  // [split][tile]
#pragma unroll 1
  for (int c0 = 0; c0 < kI8N; c0 += 8) {
    uint32_t v[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(tmem + ((uint32_t)(32 * warp) << 16) + (uint32_t)c0));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    *reinterpret_cast<int4*>(o + c0) = make_int4((int)v[0], (int)v[1], (int)v[2], (int)v[3]);
    *reinterpret_cast<int4*>(o + c0 + 4) = make_int4((int)v[4], (int)v[5], (int)v[6], (int)v[7]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kI8N));
}

// G_ij (i <= j; mirrored) = sum_{s + u <= S-1} 2^{E_i + E_j - 7 (s + u + 2)} P[(s,i),(u,j)]
// in double-double.  tile_of[I * nbt + J] = 2 (index of the tile holding
// (I, J), I <= J) + (J & 1).
__global__ void k_i8_combine(const int32_t* __restrict__ P, const int* __restrict__ tile_of, int nbt, int K, int Kp,
                             const int* __restrict__ E, double* __restrict__ Gh, double* __restrict__ Gl, int ntiles,
                             int ksplit) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)K * K) return;
  const int i = (int)(e / K), j = (int)(e % K);
  if (i > j) return;
  DD acc{0.0, 0.0};
  if (E[i] == kI8Bad || E[j] == kI8Bad) {
    acc = DD{__longlong_as_double(0x7ff8000000000000LL), 0.0};
  } else {
    for (int s = 0; s < kI8S; ++s)
      for (int u = 0; s + u <= kI8S - 1; ++u) {
        int a = s * Kp + i, b = u * Kp + j;
        if (a / kI8Tile > b / kI8Tile) {
          const int t = a;
          a = b;
          b = t;
        }
        const int I = a / kI8Tile, J = b / kI8Tile;
        const int slot = tile_of[I * nbt + J];  // 2 tile + half
        const size_t off = ((size_t)(slot >> 1) * 128 + (size_t)(a % kI8Tile)) * kI8N + (size_t)(slot & 1) * 128 +
                           (b % kI8Tile);
        int32_t v = 0;
        for (int sp = 0; sp < ksplit; ++sp) v += P[(size_t)sp * ntiles * 128 * kI8N + off];
        if (v) acc = dd_add(acc, DD{ldexp((double)v, E[i] + E[j] - 7 * (s + u + 2)), 0.0});
      }
  }
  Gh[(int64_t)i * K + j] = acc.h;
  Gl[(int64_t)i * K + j] = acc.l;
  Gh[(int64_t)j * K + i] = acc.h;
  Gl[(int64_t)j * K + i] = acc.l;
}

}  // namespace tfk
