// 32x32 diagonal-block factor+inverse: register (noinline, template-unrolled) vs smem loop.
#include <cstdio>
#include <cmath>
#include "../paper_2112_12994_b200/csrc/common.cuh"
using namespace tfk;
constexpr int LD = 36;
#define kTLD LD
__device__ __noinline__ bool diag_reg(double* dt) {
  const int m = 32, last = -1; const double floor = 0.0;
  const int lane = threadIdx.x & 31;
  double* col = dt + lane * kTLD;
  double d[32];
#pragma unroll
  for (int k = 0; k < 32; ++k) d[k] = (lane < m && k <= lane) ? col[k] : 0.0;
  bool bad = false;
  long long t0 = clock64();
  for (int i = 0; i < m; ++i) {
    double piv = __shfl_sync(0xffffffffu, d[0], i);
    if (i == last && !(piv > floor)) piv = floor;
    bad |= !(piv > 0.0) || !isfinite(piv);
    const double inv = fast_rsqrt(piv);
    const double ri = lane == i ? piv * inv : (lane > i ? d[0] * inv : 0.0);
    if (lane >= i && lane < m) col[i] = ri;
#pragma unroll
    for (int k = 1; k < 32; ++k) {
      const double rik = __shfl_sync(0xffffffffu, ri, (i + k) & 31);
      if (lane >= i + k) d[k] = fma(-rik, ri, d[k]);
    }
#pragma unroll
    for (int k = 0; k < 31; ++k) d[k] = d[k + 1];
    d[31] = 0.0;
  }
  __syncwarp();
  long long t1 = clock64();
  double xw[32];
#pragma unroll
  for (int k = 0; k < 32; ++k) xw[k] = 0.0;
  for (int i = m - 1; i >= 0; --i) {
    double a0 = (lane == i) ? 1.0 : 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll
    for (int k = 0; k < 31; k += 4) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int q = i + 1 + k + u;
        if (k + u < 31 && q < m) {
          const double rq = dt[q * kTLD + i];
          const double t = xw[k + u];
          if (u == 0) a0 = fma(-rq, t, a0);
          else if (u == 1) a1 = fma(-rq, t, a1);
          else if (u == 2) a2 = fma(-rq, t, a2);
          else a3 = fma(-rq, t, a3);
        }
      }
    }
    const double rinv = fast_rcp(dt[i * kTLD + i]);
    const double xi = lane >= i ? ((a0 + a1) + (a2 + a3)) * rinv : 0.0;
    __syncwarp();
    if (lane >= i && lane < m) col[i] = xi;
#pragma unroll
    for (int k = 31; k > 0; --k) xw[k] = xw[k - 1];
    xw[0] = xi;
    __syncwarp();
  }
  long long t2 = clock64();
  if (lane < m) for (int r = lane + 1; r < 32; ++r) col[r] = 0.0;
  if (lane == 0) printf("  factor %lld cycles, inverse %lld cycles\n", t1 - t0, t2 - t1);
  return __any_sync(0xffffffffu, bad);
}
__global__ void k(double* g, double* out, long long* cyc, int reps) {
  __shared__ double t[32 * LD];
  const int lane = threadIdx.x;
  long long tot = 0;
  for (int rep = 0; rep < reps; ++rep) {
    for (int r = 0; r < 32; ++r) t[lane * LD + r] = g[r * 32 + lane];
    __syncwarp();
    long long t0 = clock64();
    diag_reg(t);
    __syncwarp();
    tot += clock64() - t0;
  }
  for (int r = 0; r < 32; ++r) out[r * 32 + lane] = t[lane * LD + r];
  if (lane == 0) cyc[0] = tot / reps;
}
int main() {
  double G[1024], X[1024];
  for (int i = 0; i < 32; ++i) for (int j = 0; j < 32; ++j) { double s = 0; for (int t = 0; t < 64; ++t) s += sin(1.0 + i * 7 + t * 3) * sin(1.0 + j * 7 + t * 3); G[i * 32 + j] = s + (i == j ? 1.0 : 0.0); }
  double *dg, *dx; long long* dc; cudaMalloc(&dg, 8192); cudaMalloc(&dx, 8192); cudaMalloc(&dc, 64);
  cudaMemcpy(dg, G, 8192, cudaMemcpyHostToDevice);
  k<<<1, 32>>>(dg, dx, dc, 1);
  k<<<1, 32>>>(dg, dx, dc, 3);
  long long c; cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost); cudaMemcpy(X, dx, 8192, cudaMemcpyDeviceToHost);
  // check X = R^-1:  X^T G X = I  (X(r,c) stored at X[r*32+c])
  double err = 0;
  for (int i = 0; i < 32; ++i) for (int j = 0; j < 32; ++j) { double s = 0; for (int u = 0; u < 32; ++u) for (int v = 0; v < 32; ++v) s += X[u*32+i] * G[u*32+v] * X[v*32+j]; err = fmax(err, fabs(s - (i == j))); }
  printf("register diag factor+inverse: %lld cycles, err %.2e  (%s)\n", c, err, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
