// k_pass.cuh -- fused sliding-window FIR residual + leverage-score update.
//
// One launch per lag q (q = 0..p_bar), over the LSAR window rows i in [0, w):
//   s_q(i) = s_{q-1}(i) + r_{q-1}(i)^2 / R_{q-1}     (lsar.cpp:17-25; s_0 := 0)
//   r_q(i) = -y[q+i] + sum_{j=0}^{q-1} phi_q[j] * y[q-1-j+i]
//            (toeplitz.cpp:87-98: tap order j = 0..q-1 starting from -y, one
//             fma per tap -- bit-identical to the oracle's residuals())
//   per 32-row chunk:  A_c = sum s_q,  B_c = sum r_q^2   (fixed order)
//   per 2048-row tile: A_t, B_t (fixed-order tree of its chunks)
// The lag-q design matrix is never stored: each CTA stages the 2048 + q
// series values its rows touch (q-sample halo) in shared memory.
//
// k_lsar_pass (q < 16, and tf_residuals at any q): CUDA-core FIR in the
// reference's tap order; y tile in smem with one pad double every 16 (skew)
// so that the register-blocked FIR (16 consecutive outputs per thread,
// 23-value sliding window per 8 taps) reads are bank-conflict free.
// k_lsar_pass_pst (q >= 1 in the sweeps): tensor-core FIR, TMA bulk loads,
// persistent CTAs (below).
#pragma once

#include "common.cuh"

namespace tfk {

constexpr int kPassTile = 2048;
constexpr int kPassThreads = 128;
constexpr int kPassR = 16;  // outputs per thread (kPassTile / kPassThreads)
constexpr int kChunk = 32;  // rows per CDF chunk (one warp)
constexpr int kChunksPerTile = kPassTile / kChunk;

__device__ __forceinline__ int skew16(int x) { return x + (x >> 4); }

// Series window -> shared memory: eight independent loads in flight per thread
// before the stores (a load-store loop would serialise on each load's latency).
template <int NT, class F>
__device__ __forceinline__ void stage_y(double* ys, const double* src, int n, int need, F pos) {
  const int tid = threadIdx.x;
  for (int x0 = 0; x0 < n; x0 += 8 * NT) {
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int x = x0 + tid + NT * u;
      v[u] = x < need ? __ldg(src + x) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int x = x0 + tid + NT * u;
      if (x < n) ys[pos(x)] = v[u];
    }
  }
}

struct PassArgs {
  const double* y;
  int64_t w;          // window rows
  int q;              // lag of this pass (0 = initial pass: r_0 = -y[i], s_0 = 0)
  const double* phi;  // device, length q
  double* s;          // in s_{q-1}, out s_q   (length w)
  double* r;          // in r_{q-1}, out r_q   (length w)
  const double* Rprev;  // device scalar R_{q-1} (unused when q == 0)
  double* chunkA;
  double* chunkB;
  double* tileA;
  double* tileB;
  int64_t ylen;      // readable doubles at y (series + zero pad)
  // batched sweeps (k_lsar_pass only): series b = blockIdx.y reads / writes
  // every array at base + b * stride (0 for a single series)
  int64_t bs_y, bs_w, bs_chunk, bs_tile, bs_phi, bs_scal;
};

__device__ __forceinline__ void pass_batch_offset(PassArgs& a, int64_t b) {
  a.y += b * a.bs_y;
  a.s += b * a.bs_w;
  a.r += b * a.bs_w;
  a.chunkA += b * a.bs_chunk;
  a.chunkB += b * a.bs_chunk;
  a.tileA += b * a.bs_tile;
  a.tileB += b * a.bs_tile;
  a.phi += b * a.bs_phi;
  a.Rprev += b * a.bs_scal;
}


inline size_t pass_smem_bytes(int q) {
  const int phi_n = ((q + 1) & ~1) + 2;
  const int ys_n = kPassTile + q + 32;
  const int ys_sk = ys_n + (ys_n >> 4) + 2;
  const int rn_sk = kPassTile + (kPassTile >> 4) + 2;
  return sizeof(double) * (size_t)(phi_n + ys_sk + rn_sk);
}

// chunk (32 rows) and tile partial sums of s_q and r_q^2 from the tile's s_q, r_q
// in shared memory (r_q optionally in the skew16 layout): one thread per chunk, sequential over its rows from a
// rotated start (the rotation makes the strided reads conflict free); the
// tile sums are a fixed tree over the 64 chunk sums.  Deterministic; no
// per-row warp reductions.
template <bool RSKEW>
__device__ __forceinline__ void pass_partials(const PassArgs& a, const double* ss, const double* rs, int rows,
                                              int64_t i0, int64_t tile) {
  __shared__ double red[2][kChunksPerTile];
  const int tid = threadIdx.x;
  if (tid < kChunksPerTile) {
    const int c0 = kChunk * tid;
    const int nr = min(kChunk, rows - c0);
    double A = 0.0, B = 0.0;
#pragma unroll 8
    for (int k = 0; k < kChunk; ++k) {
      const int j = (k + tid) & (kChunk - 1);
      if (j < nr) {
        const double rv = rs[RSKEW ? skew16(c0 + j) : c0 + j];
        A += ss[c0 + j];
        B = fma(rv, rv, B);
      }
    }
    if (nr > 0) {
      const int64_t cidx = i0 / kChunk + tid;
      a.chunkA[cidx] = A;
      a.chunkB[cidx] = B;
    }
    red[0][tid] = A;
    red[1][tid] = B;
  }
  __syncthreads();
  if (tid < 32) {
    const double TA = warp_sum(red[0][tid] + red[0][tid + 32]);
    const double TB = warp_sum(red[1][tid] + red[1][tid + 32]);
    if (tid == 0) {
      a.tileA[tile] = TA;
      a.tileB[tile] = TB;
    }
  }
}

__global__ void __launch_bounds__(kPassThreads, 4) k_lsar_pass(PassArgs a) {
  extern __shared__ double sm[];
  if (blockIdx.y) pass_batch_offset(a, blockIdx.y);
  const int q = a.q;
  const int tid = threadIdx.x;
  const int phi_n = ((q + 1) & ~1) + 2;
  const int ys_n = kPassTile + q + 32;
  double* sphi = sm;
  double* ys = sm + phi_n;
  double* rn = ys + ys_n + (ys_n >> 4) + 2;

  const int64_t i0 = (int64_t)blockIdx.x * kPassTile;
  const int rows = (int)min((int64_t)kPassTile, a.w - i0);

  for (int t = tid; t < q; t += kPassThreads) sphi[t] = a.phi[t];
  // y[i0 .. i0 + rows + q) -- taps and targets of this tile's rows
  const int need = rows + q;
  stage_y<kPassThreads>(ys, a.y + i0, ys_n, need, [](int x) { return skew16(x); });

  __syncthreads();

  // ---- FIR: thread owns rows o = 16 tid + u ----
  double acc[kPassR];
  const int ob = kPassR * tid;
#pragma unroll
  for (int u = 0; u < kPassR; ++u) acc[u] = -ys[skew16(ob + u + q)];
  int j = 0;
  for (; j + 8 <= q; j += 8) {
    double f[8];
#pragma unroll
    for (int jj = 0; jj < 8; ++jj) f[jj] = sphi[j + jj];
    const int base = ob + q - 8 - j;  // v[k] = ys[base + k], k = 0..22
    double v[kPassR + 7];
#pragma unroll
    for (int k = 0; k < kPassR + 7; ++k) v[k] = ys[skew16(base + k)];
#pragma unroll
    for (int jj = 0; jj < 8; ++jj) {
#pragma unroll
      for (int u = 0; u < kPassR; ++u) acc[u] = fma(f[jj], v[u + 7 - jj], acc[u]);
    }
  }
  for (; j < q; ++j) {
    const double f = sphi[j];
    const int base = ob + q - 1 - j;
#pragma unroll
    for (int u = 0; u < kPassR; ++u) acc[u] = fma(f, ys[skew16(base + u)], acc[u]);
  }
#pragma unroll
  for (int u = 0; u < kPassR; ++u) rn[skew16(ob + u)] = acc[u];
  __syncthreads();

  // ---- update (coalesced), then chunk / tile partials from shared memory ----
  // previous state loaded only now: keeps the FIR's register footprint small
  // (more resident CTAs hide this latency)
  double so[kPassR], ro[kPassR];
#pragma unroll
  for (int u = 0; u < kPassR; ++u) {
    const int row = tid + kPassThreads * u;
    so[u] = 0.0;
    ro[u] = 0.0;
    if (q > 0 && row < rows) {
      so[u] = a.s[i0 + row];
      ro[u] = a.r[i0 + row];
    }
  }
  const double Rp = q > 0 ? *a.Rprev : 1.0;
  double* snew_s = ys;  // series tile is dead after the FIR barrier
#pragma unroll
  for (int u = 0; u < kPassR; ++u) {
    const int row = tid + kPassThreads * u;
    if (row < rows) {
      const double rnew = rn[skew16(row)];
      const double snew = q > 0 ? so[u] + (ro[u] * ro[u]) / Rp : 0.0;
      a.s[i0 + row] = snew;
      a.r[i0 + row] = rnew;
      snew_s[row] = snew;
    }
  }
  __syncthreads();
  pass_partials<true>(a, snew_s, rn, rows, i0, blockIdx.x);
}

// ---------------------------------------------------------------------------
// k_lsar_pass_pst: the pass for q >= 1 in the sweeps, FIR on the fp64 tensor
// cores (DMMA m8n8k4), TMA bulk loads, persistent CTAs.
//
// FIR as a polyphase GEMM: with tile rows i = 8a + b,
//   r[8a + b] = sum_k Y[a][k] Phi[k][b],   Y[a][k] = y[i0 + 8a + k]  (Hankel, stride 8)
//   Phi[k][b] = phi[q-1+b-k] for 0 <= q-1+b-k < q,  -1 for k = q + b (the target),  0 else
// so M = 256 (a), N = 8 (b), K = q + 8 per 2048-row tile; every warp owns 8
// m8 tiles (64 a-rows = 512 outputs), tile u holding a-rows 8 g + u.  The A
// fragment of tile u at k-step s equals that of tile u + 1 at step s - 2, so
// the 8 tiles walk one shared register window (one new fragment per step).
// The series tile uses the skew12 layout (x + 4 floor(x / 64): lanes 8 g + t
// read x = 64 g + t), which makes the fragment reads bank-conflict free; the
// B fragments come from a compact table phiP[j + kPhiOff] (11 distinct
// addresses per warp load, broadcast).  Summation order differs from the
// reference's tap loop (rounding ~1e-16); k_lsar_pass keeps the exact order.
//
__host__ __device__ __forceinline__ int skew12(int x) { return x + 4 * (x >> 6); }

// shared memory of k_lsar_pass_pst, in doubles:
//   [4: mbarriers][s tile: 2048][r tile: 2048][series tile: ys_sk (skew12)][phiP: phi_n]
struct PassLayout {
  int kd;     // GEMM depth: q + 8 rounded up to a k-step of 4
  int ys_n;   // series values staged per tile (2048 + kd + 8 halo)
  int ys_sk;  // their skew12 footprint (even, for 16-byte alignment)
  int phi_n;  // compact B table
  __host__ __device__ explicit PassLayout(int q) {
    kd = (q + 8 + 3) & ~3;
    ys_n = kPassTile + kd + 8;
    ys_sk = (skew12(ys_n) + 8 + 1) & ~1;
    phi_n = (q + 25) & ~1;
  }
  __host__ __device__ size_t bytes() const { return sizeof(double) * (size_t)(4 + 2 * kPassTile + ys_sk + phi_n); }
};
constexpr int kPhiOff = 16;

// DMMA FIR of one 2048-row tile (the polyphase GEMM above): ys = series tile
// (skew12), pb = phiP + kPhiOff + q - 1 + g - t; on return c0[u] / c1[u] hold
// r_q of tile rows 8 (64 warp + 8 g + u) + 2 t (+ 1)
__device__ __forceinline__ void pass_fir_acc(const double* ys, const double* pb, int nsteps, double (&c0)[8],
                                             double (&c1)[8]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int abase = 64 * warp;
#pragma unroll
  for (int u = 0; u < 8; ++u) c0[u] = c1[u] = 0.0;
  const int xbase = 8 * (abase + 8 * g) + t;
  double fe[8], fo[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    fe[u] = ys[skew12(xbase + 8 * u)];
    fo[u] = ys[skew12(xbase + 8 * u + 4)];
  }
  for (int sstep = 0; sstep < nsteps; sstep += 2) {
    const double be = pb[-4 * sstep];
#pragma unroll
    for (int u = 0; u < 8; ++u) dmma_8x8x4(c0[u], c1[u], fe[u], be);
    if (sstep + 1 < nsteps) {
      const double bo = pb[-4 * sstep - 4];
#pragma unroll
      for (int u = 0; u < 8; ++u) dmma_8x8x4(c0[u], c1[u], fo[u], bo);
    }
#pragma unroll
    for (int u = 0; u < 7; ++u) {
      fe[u] = fe[u + 1];
      fo[u] = fo[u + 1];
    }
    const int xn = xbase + 8 * 8 + 8 * (sstep >> 1);
    fe[7] = ys[skew12(xn)];
    fo[7] = ys[skew12(xn + 4)];
  }
}

// ---------------------------------------------------------------------------
// Persistent CTAs (grid = resident CTAs), each walking tiles blockIdx.x,
// + gridDim.x, ...  Loads are TMA bulk copies (cp.async.bulk + mbarrier): the
// series tile as 64-double segments into the skew12 layout, the previous
// state s_{q-1}, r_{q-1} as two contiguous copies.  The update works straight
// from the FIR accumulators, so the series buffer is free as soon as the FIR
// ends: the next tile's series copy is issued then and lands during this
// tile's update, and the next tile's state copy is issued after the update
// and lands during the next FIR.  Chunk sums: each lane folds its 8 values of
// a chunk (rows 8 a + 2 t + e), then two shuffles over t; tile sums: shuffles
// over g, fixed-order sum over the warps.  Deterministic.
__device__ __forceinline__ void pst_issue_y(const PassArgs& a, int64_t i0, double* ys, const PassLayout& L,
                                            uint64_t* bar) {  // warp 0
  const int lane = threadIdx.x & 31;
  const int ycopy = (int)min((int64_t)L.ys_n, a.ylen - i0) & ~1;
  if (lane == 0) {
    fence_proxy_async_smem();
    mbar_expect_tx(bar, (uint32_t)ycopy * 8u);
  }
  __syncwarp();
  const int nseg = (ycopy + 63) >> 6;
  for (int k = lane; k < nseg; k += 32) {
    const int len = min(64, ycopy - 64 * k);
    bulk_g2s(ys + skew12(64 * k), a.y + i0 + 64 * k, (uint32_t)len * 8u, bar);
  }
}
__device__ __forceinline__ void pst_fill_y(const PassArgs& a, int64_t i0, double* ys, const PassLayout& L) {
  const int ycopy = (int)min((int64_t)L.ys_n, a.ylen - i0) & ~1;
  for (int x = ycopy + threadIdx.x; x < L.ys_n; x += kPassThreads) ys[skew12(x)] = 0.0;
}
template <int DBG>
__device__ __forceinline__ void pst_issue_state(const PassArgs& a, int64_t i0, int rows, double* ss, double* rr,
                                                uint64_t* bar) {  // one thread
  const int rcopy = (DBG & 8) ? 0 : rows & ~1;
  fence_proxy_async_smem();
  mbar_expect_tx(bar, (uint32_t)rcopy * 16u);
  if (rcopy > 0) {
    bulk_g2s(ss, a.s + i0, (uint32_t)rcopy * 8u, bar);
    bulk_g2s(rr, a.r + i0, (uint32_t)rcopy * 8u, bar);
  }
  if (rows > rcopy && !(DBG & 8)) {  // odd last row: generic load (address not covered by the copy)
    ss[rcopy] = a.s[i0 + rcopy];
    rr[rcopy] = a.r[i0 + rcopy];
  }
}

// DBG (development, tools/pass_bench.cu; the product uses 0): bit 2 skips the
// FIR, bit 3 the state traffic
template <int DBG = 0>
__global__ void __launch_bounds__(kPassThreads, 4) k_lsar_pass_pst(PassArgs a) {
  extern __shared__ __align__(128) double sm[];
  __shared__ double red[2][kPassThreads / 32];
  const int q = a.q;
  const PassLayout L(q);
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm);  // [0]: series, [1]: state
  double* ss = sm + 4;
  double* rr = ss + kPassTile;
  double* ys = rr + kPassTile;
  double* phiP = ys + L.ys_sk;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int64_t ntile = (a.w + kPassTile - 1) / kPassTile;
  int64_t tile = blockIdx.x;
  const double invR = 1.0 / *a.Rprev;
  if (tid == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
  }
  __syncthreads();
  {
    const int64_t i0 = tile * kPassTile;
    if (warp == 0) pst_issue_y(a, i0, ys, L, &bars[0]);
    if (tid == 32) pst_issue_state<DBG>(a, i0, (int)min((int64_t)kPassTile, a.w - i0), ss, rr, &bars[1]);
    pst_fill_y(a, i0, ys, L);
  }
  for (int m = tid; m < L.phi_n; m += kPassThreads) {
    const int j = m - kPhiOff;
    phiP[m] = (j >= 0 && j < q) ? __ldg(a.phi + j) : (j == -1 ? -1.0 : 0.0);
  }
  __syncthreads();
  const double* pb = phiP + kPhiOff + q - 1 + g - t;
  const int nsteps = (DBG & 4) ? 0 : L.kd >> 2;
  for (int k = 0; tile < ntile; ++k, tile += gridDim.x) {
    const int64_t i0 = tile * kPassTile;
    const int rows = (int)min((int64_t)kPassTile, a.w - i0);
    const int64_t next = tile + gridDim.x;
    mbar_wait(&bars[0], (uint32_t)k & 1u);
    double c0[8], c1[8];
    pass_fir_acc(ys, pb, nsteps, c0, c1);
    __syncthreads();  // series tile consumed
    if (next < ntile) {
      if (warp == 0) pst_issue_y(a, next * kPassTile, ys, L, &bars[0]);
      pst_fill_y(a, next * kPassTile, ys, L);
    }
    mbar_wait(&bars[1], (uint32_t)k & 1u);
    // ---- update from the accumulators; chunk h of this lane = rows of u in [4h, 4h + 4) ----
    double A[2] = {0.0, 0.0}, B[2] = {0.0, 0.0};
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int row = 8 * (64 * warp + 8 * g + u) + 2 * t;
      if (row < rows) {
        const double2 so = *reinterpret_cast<const double2*>(ss + row);
        const double2 ro = *reinterpret_cast<const double2*>(rr + row);
        const double s0 = fma(ro.x * ro.x, invR, so.x);
        const double s1 = fma(ro.y * ro.y, invR, so.y);
        const int h = u >> 2;
        A[h] += s0;
        B[h] = fma(c0[u], c0[u], B[h]);
        if (row + 1 < rows) {
          A[h] += s1;
          B[h] = fma(c1[u], c1[u], B[h]);
          if (!(DBG & 8)) {
            *reinterpret_cast<double2*>(a.s + i0 + row) = make_double2(s0, s1);
            *reinterpret_cast<double2*>(a.r + i0 + row) = make_double2(c0[u], c1[u]);
          }
        } else if (!(DBG & 8)) {
          a.s[i0 + row] = s0;
          a.r[i0 + row] = c0[u];
        }
      }
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      A[h] += __shfl_xor_sync(0xffffffffu, A[h], 1);
      A[h] += __shfl_xor_sync(0xffffffffu, A[h], 2);
      B[h] += __shfl_xor_sync(0xffffffffu, B[h], 1);
      B[h] += __shfl_xor_sync(0xffffffffu, B[h], 2);
    }
    if (t == 0) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int c = 16 * warp + 2 * g + h;  // chunk of the tile
        if (kChunk * c < rows) {
          a.chunkA[i0 / kChunk + c] = A[h];
          a.chunkB[i0 / kChunk + c] = B[h];
        }
      }
    }
    double TA = A[0] + A[1], TB = B[0] + B[1];
#pragma unroll
    for (int o = 4; o < 32; o <<= 1) {
      TA += __shfl_xor_sync(0xffffffffu, TA, o);
      TB += __shfl_xor_sync(0xffffffffu, TB, o);
    }
    if (lane == 0) {
      red[0][warp] = TA;
      red[1][warp] = TB;
    }
    __syncthreads();  // state tile consumed; red complete
    if (tid == 0) {
      a.tileA[tile] = ((red[0][0] + red[0][1]) + red[0][2]) + red[0][3];
      a.tileB[tile] = ((red[1][0] + red[1][1]) + red[1][2]) + red[1][3];
    }
    if (tid == 32 && next < ntile)
      pst_issue_state<DBG>(a, next * kPassTile, (int)min((int64_t)kPassTile, a.w - next * kPassTile), ss, rr, &bars[1]);
  }
}

}  // namespace tfk
