// k_pass_i8.cuh -- EXPERIMENT (not in the library): the sweep's fused pass
// (FIR residual + leverage update + CDF partials, k_pass.cuh semantics) with
// the FIR on the INT8 tensor cores: an exact-product digit splitting (Ozaki
// scheme) of the fp64 series and coefficients, tcgen05.mma kind::i8 into TMEM.
// Correct (residuals within ~6 eps sum |phi y| of the fp64 DMMA pass) but
// slower than k_lsar_pass_pst below q ~ 640 on B200 (pass_i8_bench.cu,
// DESIGN.md 5): the 9 x 9 digit-plane products re-read their operands from
// shared memory (~66 KB per 32-deep K step of a 2048-row tile), and the
// four-warp epilogue (11 TMEM loads, 176 int->fp64 conversions per row block,
// the state update) does not hide behind the MMAs.
//
// Digits.  The series is scaled by a global 2^-E_y (max |y| 2^-E_y < 1/2) and
// written once per series as kPiSY signed 7-bit digit planes
//   y_t = 2^E_y sum_s dy_s(t) 2^{-7 (s+1)},  dy in [-64, 64]   (k_y_planes)
// and the lag-q FIR matrix Phi (phi taps and the -1 target tap, below) per
// launch as kPiSP planes with its own 2^E_phi (max(|phi|, 1)).  Then
//   r = sum_d 2^{E_y + E_phi - 7 (d + 2)} acc_d,   acc_d = sum_{s+u=d} sum_k dy_s dphi_u
// with acc_d exact in int32 (|dy dphi| <= 2^12, K <= 672, <= 9 plane pairs).
// Pairs with s + u > kPiL are dropped: with 63-bit planes and L = 10 the
// truncation is below the rounding of an fp64 FIR.  The
// large digit products cancel exactly in the integer sums; the final
// (L + 1)-term fp64 sum rounds at ~eps |y|, the fp64 FIR's own noise level.
//
// FIR as a polyphase GEMM, 2048-row tile i0, rows i = i0 + 16 a + b:
//   r[i] = sum_k Y[a][k] Phi[k][b],  Y[a][k] = y[i0 + 16 a + k]  (Hankel, stride 16)
//   Phi[k][b] = phi[q-1+b-k] for 0 <= q-1+b-k < q, -1 at k = q + b, 0 else
// M = 128 (a), N = 16 (b) per phi plane, K = q + 16 rounded up to 32.  The
// Hankel A operand is read straight from the staged digit bytes: a K-major
// no-swizzle UMMA descriptor with LBO = 16 B, SBO = 128 B puts row a at byte
// 16 a (core matrix (g, c) = bytes [128 g + 16 c, + 128)), so no im2col copy
// exists.  B = the Phi planes stacked along N (row 16 u + b), built once per
// CTA.  Chain s (y plane s) multiplies all phi planes u <= L - s at once
// (N = 16 min(SP, L - s + 1)) into TMEM columns [16 s, ...): column 16 d + b
// collects every pair with s + u = d.
//
// Persistent CTAs, warp-specialised: warp 4 streams the tile's 9 digit-plane
// windows (2048 + K bytes each) and its state s_{q-1}, r_{q-1} with bulk
// copies into 2-stage rings; warp 5
// issues the MMAs into one of two TMEM accumulators (176 of 256 columns each)
// and commits to the ring slot's and the accumulator's mbarriers; warps 0-3
// (TMEM lanes 0-127, thread a = rows 16 a .. 16 a + 15) drain the
// accumulator, zero it for its next use, combine, transpose the residuals
// through shared memory, apply the update
//   s_q = s_{q-1} + r_{q-1}^2 / R_{q-1}
// in place on the staged state (row 128 k + thread), write the 32-row chunk
// sums and the tile sums (fixed order) and store s, r back with bulk copies.
#pragma once

#include <cstdint>

#include "common.cuh"
#include "k_pass.cuh"

namespace tfk {

constexpr int kPiSY = 9;         // series digit planes (63 bits)
constexpr int kPiSP = 9;         // coefficient digit planes
constexpr int kPiL = 10;         // plane pairs kept: s + u <= kPiL
constexpr int kPiThreads = 224;  // warps 0-3 epilogue, 4 series loads, 5 MMA, 6 state loads
constexpr int kPiAccCols = 16 * (kPiL + 1);
constexpr int kPiMaxQ = 640;
constexpr int kPiBad = 1 << 20;
constexpr int kPiPlaneHalo = 2048 + 1024;  // readable zero bytes past the series in every plane

struct PassI8Layout {
  int K;          // GEMM depth: q + 16 rounded up to 32
  int ywin;       // staged bytes per plane and tile: 2048 + K
  int sbo;        // B operand: byte distance of 8-row groups
  size_t y_off;   // staged digit windows [2][SY][ywin]
  size_t st_off;  // staged state [2][s, r][2048] doubles (updated in place, stored back by bulk copies)
  size_t t_off;   // transposed residual tile [2048] doubles
  size_t bytes;   // dynamic shared memory (with 128 B alignment slack)
  __host__ __device__ explicit PassI8Layout(int q) {
    K = (q + 16 + 31) & ~31;
    ywin = kPassTile + K;
    sbo = (K / 16) * 128;
    y_off = ((size_t)16 * kPiSP * K + 127) & ~(size_t)127;
    st_off = (y_off + (size_t)2 * kPiSY * ywin + 127) & ~(size_t)127;
    t_off = st_off + (size_t)2 * 2 * kPassTile * sizeof(double);
    bytes = t_off + (size_t)kPassTile * sizeof(double) + 128;
  }
};

struct PassI8Args {
  PassArgs a;
  const int8_t* yp;    // digit planes, plane s at yp + s * yp_stride
  int64_t yp_stride;
  const int* ey;       // device: E_y
};

__device__ __forceinline__ uint64_t pi_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // sm_100 descriptor version; base offset 0, no swizzle
  return d;
}
__device__ __forceinline__ void pi_mma(uint32_t dtm, uint64_t da, uint64_t db, uint32_t idesc) {
  asm volatile("tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, 1;" ::"r"(dtm), "l"(da), "l"(db), "r"(idesc)
               : "memory");
}
__device__ __forceinline__ void pi_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void pi_ld16(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}
__device__ __forceinline__ void pi_st16_zero(uint32_t taddr) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(taddr),
      "r"(0u)
      : "memory");
}
__device__ __forceinline__ void pi_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void pi_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void pi_mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// byte of (row n, depth k) in a K-major no-swizzle operand with 8-row groups sbo apart
__device__ __forceinline__ int pi_lay(int n, int k, int sbo) {
  return (n >> 3) * sbo + (k >> 4) * 128 + (n & 7) * 16 + (k & 15);
}

// fixed-order pairwise sum of 16 values
__device__ __forceinline__ double pi_tree16(const double (&v)[16]) {
  double t[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) t[i] = v[2 * i] + v[2 * i + 1];
#pragma unroll
  for (int i = 0; i < 4; ++i) t[i] = t[2 * i] + t[2 * i + 1];
  return (t[0] + t[1]) + (t[2] + t[3]);
}

// max |y| and sum y^2 partials (the plane scale and the int8-pass gate)
__global__ void k_y_stats(const double* __restrict__ y, int64_t n, double* __restrict__ part) {
  __shared__ double sm[2][8];
  double m = 0.0, s2 = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double v = y[i];
    m = fmax(m, fabs(v));
    s2 = fma(v, v, s2);
  }
  for (int o = 16; o > 0; o >>= 1) {
    m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    s2 += __shfl_xor_sync(0xffffffffu, s2, o);
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    sm[0][warp] = m;
    sm[1][warp] = s2;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
      m = fmax(m, sm[0][w]);
      s2 += sm[1][w];
    }
    part[2 * blockIdx.x] = m;
    part[2 * blockIdx.x + 1] = s2;
  }
}

// digit planes of y * 2^-E_y over [0, len) (zero past n), 16 values per thread
__global__ void k_y_planes(const double* __restrict__ y, int64_t n, int64_t len, int ey, int64_t stride,
                           int8_t* __restrict__ yp) {
  const int64_t t0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 16;
  if (t0 >= len) return;
  double x[16];
#pragma unroll
  for (int u = 0; u < 16; ++u) x[u] = t0 + u < n ? ldexp(y[t0 + u], -ey) : 0.0;
#pragma unroll 1
  for (int s = 0; s < kPiSY; ++s) {
    uint32_t w[4] = {0u, 0u, 0u, 0u};
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const double v = x[u] * 128.0;  // exact
      const double d = rint(v);
      x[u] = v - d;  // exact
      w[u >> 2] |= ((uint32_t)(uint8_t)(int8_t)(int)d) << (8 * (u & 3));
    }
    *reinterpret_cast<uint4*>(yp + s * stride + t0) = make_uint4(w[0], w[1], w[2], w[3]);
  }
}

// DBG (development, tools/pass_i8_bench.cu; the product uses 0): bit 0 skips
// the MMAs, bit 1 the state traffic and the update
template <int DBG = 0>
__global__ void __launch_bounds__(kPiThreads, 1) k_lsar_pass_i8(PassI8Args args) {
  extern __shared__ __align__(128) unsigned char pism[];
  __shared__ __align__(8) uint64_t bar_yf[2], bar_ye[2], bar_af[2], bar_ae[2], bar_sf[2], bar_se[2];
  __shared__ uint32_t tmem_base;
  __shared__ double red[2][2][4];
  __shared__ int s_eph;
  const PassArgs& a = args.a;
  const int q = a.q;
  const PassI8Layout L(q);
  unsigned char* base = pism + ((128 - (smem_u32(pism) & 127)) & 127);
  unsigned char* sB = base;
  unsigned char* sY = base + L.y_off;
  double* sSt = reinterpret_cast<double*>(base + L.st_off);  // stage st: s at sSt + 4096 st, r at + 2048
  double* sT = reinterpret_cast<double*>(base + L.t_off);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t ntile = (a.w + kPassTile - 1) / kPassTile;

  if (warp == 0) {  // E_phi from max(|phi|, 1) (NaN sticks)
    double m = 1.0;
    for (int j = lane; j < q; j += 32) {
      const double v = fabs(a.phi[j]);
      m = (v > m || v != v) ? v : m;
    }
    for (int o = 16; o > 0; o >>= 1) {
      const double v = __shfl_xor_sync(0xffffffffu, m, o);
      m = (v > m || v != v) ? v : m;
    }
    if (lane == 0) {
      int e = 0;
      frexp(m, &e);
      s_eph = isfinite(m) ? e + 1 : kPiBad;
    }
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 128) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(&bar_yf[i], 1);
      mbar_init(&bar_ye[i], 1);
      mbar_init(&bar_af[i], 1);
      mbar_init(&bar_ae[i], 128);
      mbar_init(&bar_sf[i], 1);
      mbar_init(&bar_se[i], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int eph = s_eph;
  // B operand: row 16 u + b, depth k = digit u of Phi[k][b] 2^-E_phi
  for (int e = tid; e < 16 * L.K; e += kPiThreads) {
    const int k = e >> 4, b = e & 15;
    const int j = q - 1 + b - k;
    double v = (j >= 0 && j < q) ? a.phi[j] : (k == q + b ? -1.0 : 0.0);
    v = eph == kPiBad ? 0.0 : ldexp(v, -eph);
#pragma unroll
    for (int u = 0; u < kPiSP; ++u) {
      const double t = v * 128.0;
      const double d = rint(t);
      v = t - d;
      sB[pi_lay(16 * u + b, k, L.sbo)] = (unsigned char)(int8_t)(int)d;
    }
  }
  const uint32_t tmem = tmem_base;
  if (warp < 4) {  // both accumulators start at zero (every MMA accumulates)
    pi_fence_after();
    const uint32_t lanes = (uint32_t)(32 * warp) << 16;
    for (int ab = 0; ab < 2; ++ab)
      for (int c = 0; c < kPiAccCols; c += 16) pi_st16_zero(tmem + lanes + 256 * ab + c);
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  fence_proxy_async_smem();
  pi_fence_before();
  __syncthreads();
  pi_fence_after();

  if (warp == 4) {
    if (lane == 0) {  // loads: the tile's digit-plane windows
      int it = 0;
      for (int64_t tile = blockIdx.x; tile < ntile; tile += gridDim.x, ++it) {
        const int st = it & 1;
        const int64_t i0 = tile * kPassTile;
        if (it >= 2) mbar_wait(&bar_ye[st], (uint32_t)(((it >> 1) - 1) & 1));
        mbar_expect_tx(&bar_yf[st], (uint32_t)(kPiSY * L.ywin));
        for (int s = 0; s < kPiSY; ++s)
          bulk_g2s(sY + (size_t)(st * kPiSY + s) * L.ywin, args.yp + s * args.yp_stride + i0, (uint32_t)L.ywin,
                   &bar_yf[st]);
      }
    }
  } else if (warp == 6) {
    if (lane == 0) {  // loads: the tile's state s_{q-1}, r_{q-1}
      int it = 0;
      for (int64_t tile = blockIdx.x; tile < ntile; tile += gridDim.x, ++it) {
        const int st = it & 1;
        const int64_t i0 = tile * kPassTile;
        const int rows = (int)min((int64_t)kPassTile, a.w - i0);
        const int rcopy = (DBG & 2) ? 0 : rows & ~1;  // bulk sizes are multiples of 16 B; an odd last row goes direct
        if (it >= 2) mbar_wait(&bar_se[st], (uint32_t)(((it >> 1) - 1) & 1));
        mbar_expect_tx(&bar_sf[st], (uint32_t)rcopy * 16u);
        if (rcopy > 0) {
          bulk_g2s(sSt + 4096 * st, a.s + i0, (uint32_t)rcopy * 8u, &bar_sf[st]);
          bulk_g2s(sSt + 4096 * st + 2048, a.r + i0, (uint32_t)rcopy * 8u, &bar_sf[st]);
        }
      }
    }
  } else if (warp == 5) {
    if (lane == 0) {  // MMA issue: descriptors advance by 32 B (A) / 256 B (B) per K step
      const uint64_t db0 = pi_desc(smem_u32(sB), 128, (uint32_t)L.sbo);
      const int nkc = L.K / 32;
      int it = 0;
      for (int64_t tile = blockIdx.x; tile < ntile; tile += gridDim.x, ++it) {
        const int st = it & 1;
        mbar_wait(&bar_yf[st], (uint32_t)((it >> 1) & 1));
        if (it >= 2) mbar_wait(&bar_ae[st], (uint32_t)(((it >> 1) - 1) & 1));
        pi_fence_after();
        const uint32_t d0 = tmem + 256u * (uint32_t)st;
        const uint32_t ya0 = smem_u32(sY + (size_t)st * kPiSY * L.ywin);
        if (!(DBG & 1))
#pragma unroll 1
          for (int s = 0; s < kPiSY; ++s) {
            const int nu = min(kPiSP, kPiL - s + 1);
            const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(2 * nu) << 17) | (8u << 24);
            const uint32_t dt = d0 + 16u * (uint32_t)s;
            uint64_t da = pi_desc(ya0 + (uint32_t)(s * L.ywin), 16, 128), db = db0;
#pragma unroll 4
            for (int kc = 0; kc < nkc; ++kc) {
              pi_mma(dt, da, db, idesc);
              da += 2;
              db += 16;
            }
          }
        pi_commit(&bar_ye[st]);
        pi_commit(&bar_af[st]);
      }
    }
  } else if (warp < 4) {
    // epilogue.  TMEM lane a = rows 16 a .. 16 a + 15: combine the digit sums,
    // transpose through shared memory (16-byte slots XOR-swizzled by a & 7:
    // conflict-free both ways), then the update in the coalesced mapping
    // row = 128 k + tid on the staged state, 32-row chunk = one warp, stored
    // back by bulk copies.
    const int ar = tid;
    const double invR = 1.0 / *a.Rprev;
    const int ey = *args.ey;
    double scale[kPiL + 1];
#pragma unroll
    for (int d = 0; d <= kPiL; ++d) scale[d] = ldexp(1.0, ey + eph - 7 * (d + 2));
    const uint32_t lanes = (uint32_t)(32 * warp) << 16;
    int it = 0;
    for (int64_t tile = blockIdx.x; tile < ntile; tile += gridDim.x, ++it) {
      const int ab = it & 1, st = it & 1;
      const int64_t i0 = tile * kPassTile;
      const int rows = (int)min((int64_t)kPassTile, a.w - i0);
      mbar_wait(&bar_af[ab], (uint32_t)((it >> 1) & 1));
      pi_fence_after();
      double rv[16];
#pragma unroll
      for (int b = 0; b < 16; ++b) rv[b] = 0.0;
#pragma unroll
      for (int d = kPiL; d >= 0; --d) {  // small terms first
        uint32_t v[16];
        pi_ld16(tmem + lanes + 256u * ab + 16u * d, v);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int b = 0; b < 16; ++b) rv[b] = fma((double)(int)v[b], scale[d], rv[b]);
      }
#pragma unroll
      for (int c = 0; c < kPiAccCols; c += 16) pi_st16_zero(tmem + lanes + 256u * ab + c);
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      pi_fence_before();
      pi_mbar_arrive(&bar_ae[ab]);
      if (eph == kPiBad) {
#pragma unroll
        for (int b = 0; b < 16; ++b) rv[b] = __longlong_as_double(0x7ff8000000000000LL);
      }
      if (tid == 0 && it >= 1) {  // the previous tile's bulk stores have read their stage: release it to the loader
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        pi_mbar_arrive(&bar_se[st ^ 1]);
      }
      // transpose: double2 v of row block a at slot v ^ (a & 7)
#pragma unroll
      for (int v = 0; v < 8; ++v)
        reinterpret_cast<double2*>(sT)[8 * ar + (v ^ (ar & 7))] = make_double2(rv[2 * v], rv[2 * v + 1]);
      mbar_wait(&bar_sf[st], (uint32_t)((it >> 1) & 1));
      asm volatile("bar.sync 1, 128;" ::: "memory");  // sT complete
      double* ss = sSt + 4096 * st;
      double* rr = ss + 2048;
      double TA = 0.0, TB = 0.0;
      if (!(DBG & 2)) {
        const bool odd = rows & 1;
#pragma unroll 4
        for (int k = 0; k < 16; ++k) {
          const int i = 128 * k + tid;
          const int ra = i >> 4, rb = i & 15;
          const double rnew = sT[16 * ra + 2 * ((rb >> 1) ^ (ra & 7)) + (rb & 1)];
          double A = 0.0, B = 0.0;
          if (i < rows) {
            const bool direct = odd && i == rows - 1;  // not covered by the bulk copies
            const double so = direct ? a.s[i0 + i] : ss[i];
            const double ro = direct ? a.r[i0 + i] : rr[i];
            const double sn = fma(ro * ro, invR, so);
            if (direct) {
              a.s[i0 + i] = sn;
              a.r[i0 + i] = rnew;
            } else {
              ss[i] = sn;
              rr[i] = rnew;
            }
            A = sn;
            B = rnew * rnew;
          }
          A = warp_sum(A);
          B = warp_sum(B);
          const int c = 4 * k + warp;  // chunk of the tile
          if (lane == 0 && kChunk * c < rows) {
            a.chunkA[i0 / kChunk + c] = A;
            a.chunkB[i0 / kChunk + c] = B;
          }
          TA += A;
          TB += B;
        }
      }
      if (lane == 0) {
        red[ab][0][warp] = TA;
        red[ab][1][warp] = TB;
      }
      fence_proxy_async_smem();  // the state writes, before the bulk stores read them
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (tid == 0) {
        a.tileA[tile] = ((red[ab][0][0] + red[ab][0][1]) + red[ab][0][2]) + red[ab][0][3];
        a.tileB[tile] = ((red[ab][1][0] + red[ab][1][1]) + red[ab][1][2]) + red[ab][1][3];
        const int rcopy = (DBG & 2) ? 0 : rows & ~1;
        if (rcopy > 0) {
          bulk_s2g(a.s + i0, ss, (uint32_t)rcopy * 8u);
          bulk_s2g(a.r + i0, rr, (uint32_t)rcopy * 8u);
        }
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
    }
    if (tid == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  pi_fence_before();
  __syncthreads();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

}  // namespace tfk
