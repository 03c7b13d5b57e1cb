#include <cstdio>
__global__ void shfl_tput(double* out, int iters) {
  double v[8]; for (int k = 0; k < 8; ++k) v[k] = threadIdx.x + k;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = __shfl_sync(0xffffffffu, v[k], (threadIdx.x + k + i) & 31);
  }
  long long t1 = clock64();
  double s = 0; for (int k = 0; k < 8; ++k) s += v[k];
  if (threadIdx.x == 0) { out[0] = (double)(t1 - t0) / (iters * 8.0); }
  if (s == 1234.5) out[1] = s;
}
__global__ void lds_bcast_tput(double* out, int iters) {
  __shared__ double buf[64];
  if (threadIdx.x < 64) buf[threadIdx.x] = threadIdx.x;
  __syncwarp();
  double v[8] = {};
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] += buf[(i + k) & 63];
  }
  long long t1 = clock64();
  double s = 0; for (int k = 0; k < 8; ++k) s += v[k];
  if (threadIdx.x == 0) out[2] = (double)(t1 - t0) / (iters * 8.0);
  if (s == 1234.5) out[3] = s;
}
__global__ void dfma_tput1(double* out, int iters) {
  double v[8]; for (int k = 0; k < 8; ++k) v[k] = threadIdx.x + k;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = fma(v[k], 0.999, 1e-3);
  }
  long long t1 = clock64();
  double s = 0; for (int k = 0; k < 8; ++k) s += v[k];
  if (threadIdx.x == 0) out[4] = (double)(t1 - t0) / (iters * 8.0);
  if (s == 1234.5) out[5] = s;
}
__global__ void mov_tput(double* out, int iters) {
  double v[32]; for (int k = 0; k < 32; ++k) v[k] = threadIdx.x + k;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    double t = v[0];
#pragma unroll
    for (int k = 0; k < 31; ++k) v[k] = v[k + 1];
    v[31] = t + 1.0;
  }
  long long t1 = clock64();
  double s = 0; for (int k = 0; k < 32; ++k) s += v[k];
  if (threadIdx.x == 0) out[6] = (double)(t1 - t0) / iters;
  if (s == 1234.5) out[7] = s;
}
int main() {
  double* d; cudaMalloc(&d, 64 * 8); double h[8];
  shfl_tput<<<1, 32>>>(d, 1000); lds_bcast_tput<<<1, 32>>>(d, 1000); dfma_tput1<<<1, 32>>>(d, 1000); mov_tput<<<1,32>>>(d, 1000);
  cudaMemcpy(h, d, 64, cudaMemcpyDeviceToHost);
  printf("1 warp: SHFL.64 %.1f cyc/op, LDS.64 bcast %.1f cyc/op, DFMA %.1f cyc/op, 32-reg rotate %.1f cyc/iter\n", h[0], h[2], h[4], h[6]);
  return 0;
}
