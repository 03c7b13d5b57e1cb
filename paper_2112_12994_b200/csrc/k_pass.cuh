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
  for (int x = tid; x < ys_n; x += kPassThreads)
    ys[skew16(x)] = x < need ? __ldg(a.y + i0 + x) : 0.0;

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

}  // namespace tfk
