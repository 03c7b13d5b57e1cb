// fir_dfma_vs_dmma.cu -- the north star's "tensor cores only where ncu shows
// they beat fp64 FMA" check for the fused pass's FIR: at lags q in {16, 64,
// 100, 200, 500} over w = 1e7 rows, the register-blocked CUDA-core DFMA pass
// (k_lsar_pass: 16 outputs per thread, the reference's tap order) against
// the DMMA pass (k_lsar_pass_pst: polyphase m8n8k4 fp64 tensor-core GEMM,
// persistent, TMA-fed).  Same inputs, same outputs (s, r, chunk/tile sums).
// Prints CUDA-event times; run under ncu for the pipe metrics
// (profiles/r02_fir_dfma_vs_dmma.txt).
// build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I paper_2112_12994_b200/csrc tools/fir_dfma_vs_dmma.cu -o tools/bin/fir_dfma_vs_dmma
#include <cuda_runtime.h>
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>
#include "k_pass.cuh"
using namespace tfk;
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s line %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)
int main(int argc, char** argv) {
  const int reps = argc > 1 ? atoi(argv[1]) : 10;
  const int64_t w = 10000000, n = w + 600;
  std::vector<double> hy(n + 64);
  std::mt19937_64 g(1);
  std::normal_distribution<double> nd;
  for (auto& v : hy) v = nd(g);
  double *y, *s, *r, *cA, *cB, *tA, *tB, *phi, *R;
  CK(cudaMalloc(&y, sizeof(double) * hy.size()));
  CK(cudaMemcpy(y, hy.data(), sizeof(double) * hy.size(), cudaMemcpyHostToDevice));
  CK(cudaMalloc(&s, sizeof(double) * w));
  CK(cudaMalloc(&r, sizeof(double) * w));
  CK(cudaMemcpy(s, hy.data(), sizeof(double) * w, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(r, hy.data() + 1, sizeof(double) * w, cudaMemcpyHostToDevice));
  CK(cudaMalloc(&cA, sizeof(double) * (w / 32 + 2)));
  CK(cudaMalloc(&cB, sizeof(double) * (w / 32 + 2)));
  const int64_t ntile = (w + kPassTile - 1) / kPassTile;
  CK(cudaMalloc(&tA, sizeof(double) * ntile));
  CK(cudaMalloc(&tB, sizeof(double) * ntile));
  std::vector<double> hp(1024);
  for (auto& v : hp) v = 0.01 * nd(g);
  CK(cudaMalloc(&phi, sizeof(double) * 1024));
  CK(cudaMemcpy(phi, hp.data(), sizeof(double) * 1024, cudaMemcpyHostToDevice));
  CK(cudaMalloc(&R, sizeof(double)));
  const double one = 1.0;
  CK(cudaMemcpy(R, &one, sizeof(double), cudaMemcpyHostToDevice));
  PassArgs a{};
  a.y = y; a.w = w; a.phi = phi; a.s = s; a.r = r; a.Rprev = R;
  a.chunkA = cA; a.chunkB = cB; a.tileA = tA; a.tileB = tB; a.ylen = n + 64;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto timeit = [&](auto launch) {
    for (int i = 0; i < 2; ++i) launch();
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    for (int i = 0; i < reps; ++i) launch();
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    return ms * 1e3 / reps;
  };
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  printf("w = %lld rows; FIR flops per launch = 2 (q + 1) w; state traffic 40 B/row\n", (long long)w);
  for (int q : {16, 64, 100, 200, 500}) {
    a.q = q;
    const double fl = 2.0 * (q + 1) * w;
    const size_t sm0 = pass_smem_bytes(q);
    CK(cudaFuncSetAttribute(k_lsar_pass, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm0));
    const double t_dfma = timeit([&] { k_lsar_pass<<<(unsigned)ntile, kPassThreads, sm0>>>(a); });
    const size_t smp = PassLayout(q).bytes();
    CK(cudaFuncSetAttribute(k_lsar_pass_pst<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smp));
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_lsar_pass_pst<0>, kPassThreads, smp);
    const unsigned grid = (unsigned)std::min<int64_t>(ntile, (int64_t)occ * nsm);
    const double t_dmma = timeit([&] { k_lsar_pass_pst<0><<<grid, kPassThreads, smp>>>(a); });
    CK(cudaGetLastError());
    printf("q=%3d  DFMA k_lsar_pass %8.1f us (%5.1f TF/s)   DMMA k_lsar_pass_pst %8.1f us (%5.1f TF/s)   DMMA/DFMA speedup %.2fx\n",
           q, t_dfma, fl / t_dfma / 1e6, t_dmma, fl / t_dmma / 1e6, t_dfma / t_dmma);
  }
  return 0;
}
