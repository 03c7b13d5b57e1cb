// k_pass.cuh -- fused sliding-window FIR residual + leverage-score update.
//
// One launch per lag q (q = 0..p_bar), over the LSAR window rows i in [0, w):
//   s_q(i) = s_{q-1}(i) + r_{q-1}(i)^2 / R_{q-1}     (lsar.cpp:17-25; s_0 := 0)
//   r_q(i) = -y[q+i] + sum_{j=0}^{q-1} phi_q[j] * y[q-1-j+i]
//            (toeplitz.cpp:87-98: tap order j = 0..q-1 starting from -y, one
//             fma per tap -- bit-identical to the oracle's residuals())
//   per 32-row chunk:  A_c = sum s_q,  B_c = sum r_q^2   (fixed-order warp tree)
//   per 2048-row tile: A_t, B_t (fixed-order sum of its chunks)
// The lag-q design matrix is never stored: each CTA stages the 2048 + q
// series values its rows touch (q-sample halo) in shared memory.
//
// Layout: y tile in smem with one pad double every 16 (skew) so that the
// register-blocked FIR (16 consecutive outputs per thread, 23-value sliding
// window per 8 taps) reads are bank-conflict free.
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
};

inline size_t pass_smem_bytes(int q) {
  const int phi_n = ((q + 1) & ~1) + 2;
  const int ys_n = kPassTile + q + 32;
  const int ys_sk = ys_n + (ys_n >> 4) + 2;
  const int rn_sk = kPassTile + (kPassTile >> 4) + 2;
  return sizeof(double) * (size_t)(phi_n + ys_sk + rn_sk);
}

__global__ void __launch_bounds__(kPassThreads, 4) k_lsar_pass(PassArgs a) {
  extern __shared__ double sm[];
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

  // ---- update + chunk partials (coalesced: warp covers one 32-row chunk per u) ----
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
  const int warp = tid >> 5, lane = tid & 31;
  double tA = 0.0, tB = 0.0;
#pragma unroll
  for (int u = 0; u < kPassR; ++u) {
    const int row = tid + kPassThreads * u;
    double snew = 0.0, rnew = 0.0;
    if (row < rows) {
      rnew = rn[skew16(row)];
      snew = q > 0 ? so[u] + (ro[u] * ro[u]) / Rp : 0.0;
      a.s[i0 + row] = snew;
      a.r[i0 + row] = rnew;
    }
    const double cA = warp_sum(snew);
    const double cB = warp_sum(rnew * rnew);
    const int crow = kPassThreads * u + kChunk * warp;  // chunk's first row in tile
    if (lane == 0 && crow < rows) {
      const int64_t cidx = (i0 + crow) / kChunk;
      a.chunkA[cidx] = cA;
      a.chunkB[cidx] = cB;
    }
    tA += cA;
    tB += cB;
  }
  __shared__ double wA[kPassThreads / 32], wB[kPassThreads / 32];
  if (lane == 0) {
    wA[warp] = tA;
    wB[warp] = tB;
  }
  __syncthreads();
  if (tid == 0) {
    a.tileA[blockIdx.x] = ((wA[0] + wA[1]) + wA[2]) + wA[3];
    a.tileB[blockIdx.x] = ((wB[0] + wB[1]) + wB[2]) + wB[3];
  }
}


// ---------------------------------------------------------------------------
// Tensor-core variant of the fused pass for larger lags (fp64 DMMA m8n8k4).
// The FIR over a tile is a polyphase GEMM: with rows i = 8a + b,
//   r[8a + b] = sum_k Y[a][k] Phi[k][b],   Y[a][k] = y[i0 + 8a + k]  (Hankel, stride 8)
//   Phi[k][b] = phi[q-1+b-k] for 0 <= q-1+b-k < q,  -1 for k = q + b  (the target),  0 else
// so M = 256 (a), N = 8 (b), K = q + 8 per 2048-row tile; every warp owns 8
// m8 tiles (64 a-rows = 512 outputs), tile u holding a-rows 8 g + u.  Then the
// A fragment of tile u at k-step s equals that of tile u + 1 at step s - 2, so
// the 8 tiles walk one shared register window (one new fragment per step).  The y tile
// uses a padded layout (x + 4 floor(x / 64): lanes 8 g + t read x = 64 g + t)
// that makes the fragment reads bank-conflict free; Phi fragments are tabulated once per CTA.
// Summation order differs from the reference's tap loop (rounding ~1e-16);
// the exact-order FMA kernel above serves tf_residuals and small lags.
__host__ __device__ __forceinline__ int skew12(int x) { return x + 4 * (x >> 6); }

inline int pass_mma_kd(int q) { return (q + 8 + 3) & ~3; }
inline size_t pass_mma_smem_bytes(int q) {
  const int kd = pass_mma_kd(q);
  const int ys_n = kPassTile + kd + 8;
  const int ys_sk = skew12(ys_n) + 8;
  const int rn_sk = kPassTile + (kPassTile >> 4) + 2;
  return sizeof(double) * (size_t)(kd * 8 + ys_sk + rn_sk);
}

__global__ void __launch_bounds__(kPassThreads, 5) k_lsar_pass_mma(PassArgs a) {
  extern __shared__ double sm[];
  const int q = a.q;
  const int kd = (q + 8 + 3) & ~3;
  const int ys_n = kPassTile + kd + 8;
  double* phiF = sm;                       // [kd / 4][32]: B fragment of k-step s for each lane
  double* ys = sm + kd * 8;
  double* rn = ys + skew12(ys_n) + 8;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t i0 = (int64_t)blockIdx.x * kPassTile;
  const int rows = (int)min((int64_t)kPassTile, a.w - i0);
  const int need = rows + q;
  stage_y<kPassThreads>(ys, a.y + i0, ys_n, need, [](int x) { return skew12(x); });
  for (int e = tid; e < kd * 8; e += kPassThreads) {
    const int sstep = e >> 5, ln = e & 31;
    const int k = 4 * sstep + (ln & 3), b = ln >> 2;
    const int j = q - 1 + b - k;
    phiF[e] = (j >= 0 && j < q) ? __ldg(a.phi + j) : (k == q + b ? -1.0 : 0.0);
  }
  __syncthreads();
  // ---- FIR on DMMA: warp tiles a in [64 warp, 64 warp + 64) ----
  const int g = lane >> 2, t = lane & 3;
  const int abase = 64 * warp;
  double c0[8], c1[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) c0[u] = c1[u] = 0.0;
  // m8 tile u holds a-rows abase + 8 g + u (g = lane / 4), so its A fragment at
  // k-step s is f[s + 2u] with f[m] = Y[abase + 8 g][4 m + t]
  const int xbase = 8 * (abase + 8 * g) + t;
  double fe[8], fo[8];  // windows for even / odd steps: fe[u] = f[s + 2u] (s even)
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    fe[u] = ys[skew12(xbase + 8 * u)];      // f[2u]     (step 0)
    fo[u] = ys[skew12(xbase + 8 * u + 4)];  // f[2u + 1] (step 1)
  }
  const int nsteps = kd >> 2;
  for (int sstep = 0; sstep < nsteps; sstep += 2) {
    const double be = phiF[sstep * 32 + lane];
#pragma unroll
    for (int u = 0; u < 8; ++u) dmma_8x8x4(c0[u], c1[u], fe[u], be);
    if (sstep + 1 < nsteps) {
      const double bo = phiF[(sstep + 1) * 32 + lane];
#pragma unroll
      for (int u = 0; u < 8; ++u) dmma_8x8x4(c0[u], c1[u], fo[u], bo);
    }
    // advance both windows by one tile: f[s + 2 + 2u] = old window[u + 1]
#pragma unroll
    for (int u = 0; u < 7; ++u) {
      fe[u] = fe[u + 1];
      fo[u] = fo[u + 1];
    }
    const int xn = xbase + 8 * 8 + 8 * (sstep >> 1);  // f[sstep + 2 + 14] = Y[.][4 (sstep + 16) + t]
    fe[7] = ys[skew12(xn)];
    fo[7] = ys[skew12(xn + 4)];
  }
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const int r = 8 * (abase + 8 * g + u) + 2 * t;
    rn[skew16(r)] = c0[u];
    rn[skew16(r + 1)] = c1[u];
  }
  __syncthreads();
  // ---- update + chunk partials (identical to k_lsar_pass) ----
  double so[kPassR], ro[kPassR];
#pragma unroll
  for (int u = 0; u < kPassR; ++u) {
    const int row = tid + kPassThreads * u;
    so[u] = 0.0;
    ro[u] = 0.0;
    if (row < rows) {
      so[u] = a.s[i0 + row];
      ro[u] = a.r[i0 + row];
    }
  }
  const double Rp = *a.Rprev;
  double tA = 0.0, tB = 0.0;
#pragma unroll
  for (int u = 0; u < kPassR; ++u) {
    const int row = tid + kPassThreads * u;
    double snew = 0.0, rnew = 0.0;
    if (row < rows) {
      rnew = rn[skew16(row)];
      snew = so[u] + (ro[u] * ro[u]) / Rp;
      a.s[i0 + row] = snew;
      a.r[i0 + row] = rnew;
    }
    const double cA = warp_sum(snew);
    const double cB = warp_sum(rnew * rnew);
    const int crow = kPassThreads * u + kChunk * warp;
    if (lane == 0 && crow < rows) {
      const int64_t cidx = (i0 + crow) / kChunk;
      a.chunkA[cidx] = cA;
      a.chunkB[cidx] = cB;
    }
    tA += cA;
    tB += cB;
  }
  __shared__ double wA[kPassThreads / 32], wB[kPassThreads / 32];
  if (lane == 0) {
    wA[warp] = tA;
    wB[warp] = tB;
  }
  __syncthreads();
  if (tid == 0) {
    a.tileA[blockIdx.x] = ((wA[0] + wA[1]) + wA[2]) + wA[3];
    a.tileB[blockIdx.x] = ((wB[0] + wB[1]) + wB[2]) + wB[3];
  }
}

}  // namespace tfk
