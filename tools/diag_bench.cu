// 32x32 diagonal-block factor+inverse: register (noinline, template-unrolled) vs smem loop.
#include <cstdio>
#include <cmath>
#include "../paper_2112_12994_b200/csrc/common.cuh"
using namespace tfk;
constexpr int LD = 36;
template <int I> struct F { static __device__ __forceinline__ void run(double (&d)[32], int lane, bool& bad) {
    const double piv = __shfl_sync(0xffffffffu, d[I], I);
    bad |= !(piv > 0.0);
    const double inv = fast_rsqrt(piv);
    if (lane == I) d[I] = piv * inv; else if (lane > I) d[I] *= inv;
#pragma unroll
    for (int r = I + 1; r < 32; ++r) { const double rir = __shfl_sync(0xffffffffu, d[I], r); if (lane >= r) d[r] = fma(-rir, d[I], d[r]); }
    F<I + 1>::run(d, lane, bad); } };
template <> struct F<32> { static __device__ __forceinline__ void run(double (&)[32], int, bool&) {} };
template <int I> struct V { static __device__ __forceinline__ void run(double (&d)[32], int lane) {
    double acc = (lane == I) ? 1.0 : 0.0;
#pragma unroll
    for (int q = I + 1; q < 32; ++q) { const double riq = __shfl_sync(0xffffffffu, d[I], q); if (lane >= q) acc = fma(-riq, d[q], acc); }
    const double rinv = fast_rcp(__shfl_sync(0xffffffffu, d[I], I));
    d[I] = lane >= I ? acc * rinv : 0.0;
    V<I - 1>::run(d, lane); } };
template <> struct V<-1> { static __device__ __forceinline__ void run(double (&)[32], int) {} };
__device__ __noinline__ bool diag_reg(double* dt) {
  const int lane = threadIdx.x & 31;
  double d[32];
#pragma unroll
  for (int r = 0; r < 32; ++r) d[r] = r <= lane ? dt[lane * LD + r] : 0.0;
  bool bad = false;
  F<0>::run(d, lane, bad);
  V<31>::run(d, lane);
#pragma unroll
  for (int r = 0; r < 32; ++r) dt[lane * LD + r] = r <= lane ? d[r] : 0.0;
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
  k<<<1, 32>>>(dg, dx, dc, 20);
  long long c; cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost); cudaMemcpy(X, dx, 8192, cudaMemcpyDeviceToHost);
  // check X = R^-1:  X^T G X = I  (X(r,c) stored at X[r*32+c])
  double err = 0;
  for (int i = 0; i < 32; ++i) for (int j = 0; j < 32; ++j) { double s = 0; for (int u = 0; u < 32; ++u) for (int v = 0; v < 32; ++v) s += X[u*32+i] * G[u*32+v] * X[v*32+j]; err = fmax(err, fabs(s - (i == j))); }
  printf("register diag factor+inverse: %lld cycles, err %.2e  (%s)\n", c, err, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
