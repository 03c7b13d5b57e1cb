// Microbenchmarks: DMMA latency/throughput, register vs smem 32x32 Cholesky.
#include <cstdio>
#include "../paper_2112_12994_b200/csrc/common.cuh"
using namespace tfk;

__global__ void dmma_lat(double* out, int iters) {
  double c0 = 0, c1 = 0, a = threadIdx.x * 1e-3, b = 1.0;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) dmma_8x8x4(c0, c1, a, b);  // dependent chain
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = (double)(t1 - t0) / iters;
  if (c0 == 1234.5) out[1] = c1;
}
__global__ void dmma_tput(double* out, int iters) {
  double c[8][2] = {}; double a = threadIdx.x * 1e-3, b = 1.0;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) dmma_8x8x4(c[k][0], c[k][1], a, b);
  }
  long long t1 = clock64();
  __shared__ double s[32];
  if (threadIdx.x % 32 == 0) s[threadIdx.x / 32] = (double)(t1 - t0);
  __syncthreads();
  if (threadIdx.x == 0) out[2] = s[0] / (iters * 8.0);  // cycles per DMMA per warp
  double acc = 0; for (int k = 0; k < 8; ++k) acc += c[k][0] + c[k][1];
  if (acc == 1234.5) out[3] = acc;
}
__global__ void dfma_lat(double* out, int iters) {
  double a = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) a = fma(a, 0.999, 1e-3);
  long long t1 = clock64();
  if (threadIdx.x == 0) out[4] = (double)(t1 - t0) / iters;
  if (a == 1234.5) out[5] = a;
}
__global__ void lds_lat(double* out, int iters) {
  __shared__ int s[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) s[i] = (i + 1) & 1023;
  __syncthreads();
  int p = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) p = s[p];
  long long t1 = clock64();
  if (threadIdx.x == 0) out[6] = (double)(t1 - t0) / iters;
  if (p == 12345) out[7] = p;
}
__global__ void shfl_lat(double* out, int iters) {
  double v = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) v = __shfl_sync(0xffffffffu, v, (threadIdx.x + 1) & 31) + 1.0;
  long long t1 = clock64();
  if (threadIdx.x == 0) out[8] = (double)(t1 - t0) / iters;
  if (v == 12345) out[9] = v;
}
int main() {
  double* d; cudaMalloc(&d, 64 * sizeof(double));
  double h[16] = {};
  dmma_lat<<<1, 32>>>(d, 1000); dmma_tput<<<1, 32>>>(d, 1000);
  dfma_lat<<<1, 32>>>(d, 1000); lds_lat<<<1, 32>>>(d, 1000); shfl_lat<<<1, 32>>>(d, 1000);
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("DMMA latency %.1f cyc, 1-warp DMMA issue %.1f cyc/DMMA, DFMA latency %.1f, LDS latency %.1f, SHFL+DADD %.1f\n", h[0], h[2], h[4], h[6], h[8]);
  for (int w : {1, 2, 4, 8, 16, 32}) {
    dmma_tput<<<1, 32 * w>>>(d, 1000); cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("  %2d warps: %.1f cycles per DMMA per warp -> %.1f FMA/clk/SM\n", w, h[2], 256.0 * w / h[2]);
  }
  return 0;
}
