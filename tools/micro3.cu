#include <cstdio>
#include <cmath>
#include "../paper_2112_12994_b200/csrc/common.cuh"
using namespace tfk;
constexpr int LD = 36;
// variant A: shuffle broadcast of the scaled pivot row
__device__ __forceinline__ void factA(double* dt, double* rb) {
  const int lane = threadIdx.x & 31; const int m = 32;
  double* col = dt + lane * LD;
  double d[32];
#pragma unroll
  for (int k = 0; k < 32; ++k) d[k] = (k <= lane) ? col[k] : 0.0;
  for (int i = 0; i < m; ++i) {
    double piv = __shfl_sync(0xffffffffu, d[0], i);
    const double inv = fast_rsqrt(piv);
    const double ri = lane == i ? piv * inv : (lane > i ? d[0] * inv : 0.0);
    if (lane >= i) col[i] = ri;
#pragma unroll
    for (int k = 1; k < 32; ++k) {
      const double rik = __shfl_sync(0xffffffffu, ri, (i + k) & 31);
      if (lane >= i + k) d[k] = fma(-rik, ri, d[k]);
    }
#pragma unroll
    for (int k = 0; k < 31; ++k) d[k] = d[k + 1];
    d[31] = 0.0;
  }
}
// variant B: pivot row published to shared memory, read back by broadcast
__device__ __forceinline__ void factB(double* dt, double* rb) {
  const int lane = threadIdx.x & 31; const int m = 32;
  double* col = dt + lane * LD;
  double d[32];
#pragma unroll
  for (int k = 0; k < 32; ++k) d[k] = (k <= lane) ? col[k] : 0.0;
  for (int i = 0; i < m; ++i) {
    const double piv = __shfl_sync(0xffffffffu, d[0], i);
    const double inv = fast_rsqrt(piv);
    const double ri = lane == i ? piv * inv : (lane > i ? d[0] * inv : 0.0);
    rb[lane] = ri;  // row i of R, published
    if (lane >= i) col[i] = ri;
    __syncwarp();
#pragma unroll
    for (int k = 1; k < 32; ++k) {
      const double rik = rb[(i + k) & 31];
      if (lane >= i + k) d[k] = fma(-rik, ri, d[k]);
    }
    __syncwarp();
#pragma unroll
    for (int k = 0; k < 31; ++k) d[k] = d[k + 1];
    d[31] = 0.0;
  }
}
template <int V>
__global__ void kk(const double* g, double* out, long long* cyc) {
  __shared__ double t[32 * LD]; __shared__ double rb[32];
  const int lane = threadIdx.x;
  long long best = 1LL << 60;
  for (int rep = 0; rep < 5; ++rep) {
    for (int r = 0; r < 32; ++r) t[lane * LD + r] = g[r * 32 + lane];
    __syncwarp();
    long long t0 = clock64();
    if (V == 0) factA(t, rb); else factB(t, rb);
    __syncwarp();
    long long dt = clock64() - t0; if (dt < best) best = dt;
  }
  for (int r = 0; r < 32; ++r) out[r * 32 + lane] = t[lane * LD + r];
  if (lane == 0) cyc[V] = best;
}
int main() {
  double G[1024];
  for (int i = 0; i < 32; ++i) for (int j = 0; j < 32; ++j) { double s = 0; for (int t = 0; t < 64; ++t) s += sin(1.0 + i * 7 + t * 3) * sin(1.0 + j * 7 + t * 3); G[i * 32 + j] = s + (i == j ? 1.0 : 0.0); }
  double *dg, *dx; long long* dc; cudaMalloc(&dg, 8192); cudaMalloc(&dx, 8192); cudaMalloc(&dc, 64);
  cudaMemcpy(dg, G, 8192, cudaMemcpyHostToDevice);
  kk<0><<<1, 32>>>(dg, dx, dc); kk<1><<<1, 32>>>(dg, dx, dc);
  long long c[2]; cudaMemcpy(c, dc, 16, cudaMemcpyDeviceToHost);
  printf("32x32 factor: shuffle-broadcast %lld cycles, smem-broadcast %lld cycles (%s)\n", c[0], c[1], cudaGetErrorString(cudaGetLastError()));
  return 0;
}
