// pass_bench.cu -- the fused LSAR pass kernels in isolation (development helper).
// Times k_lsar_pass and k_lsar_pass_tma over w = 1e7 rows at several lags,
// the latter also with its debug switches (dbg bit 2: no FIR, bit 3: no state
// traffic) to split the cost into memory and FIR parts, plus per-CTA phase
// timestamps (%globaltimer).
// build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I paper_2112_12994_b200/csrc tools/pass_bench.cu -o gpurun_out/pass_bench
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <random>
#include <algorithm>
#include "k_pass.cuh"
using namespace tfk;
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s line %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)
int main() {
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
  const int reps = 20;
  auto timeit = [&](auto launch) {
    for (int i = 0; i < 3; ++i) launch();
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    for (int i = 0; i < reps; ++i) launch();
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    return ms * 1e3 / reps;
  };
  for (int q : {1, 8, 15}) {  // CUDA-core pass (exact tap order)
    a.q = q;
    a.dbg = 0;
    const size_t sm0 = pass_smem_bytes(q);
    CK(cudaFuncSetAttribute(k_lsar_pass, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm0));
    const double t = timeit([&] { k_lsar_pass<<<(unsigned)ntile, kPassThreads, sm0>>>(a); });
    CK(cudaGetLastError());
    printf("q=%3d k_lsar_pass %7.1f us  %.0f GB/s (40 B/row moved)\n", q, t, 40.0 * w / t / 1e3);
  }
  for (int q : {16, 50, 100, 200, 500}) {
    a.q = q;
    const size_t sm2 = PassTmaLayout(q).bytes();
    CK(cudaFuncSetAttribute(k_lsar_pass_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm2));
    int o2 = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o2, k_lsar_pass_tma, kPassThreads, sm2);
    double t_tma[4];
    for (int m = 0; m < 4; ++m) {
      a.dbg = 4 * m;
      t_tma[m] = timeit([&] { k_lsar_pass_tma<<<(unsigned)ntile, kPassThreads, sm2>>>(a); });
    }
    a.dbg = 0;
    CK(cudaGetLastError());
    const double fl = 2.0 * (q + 1) * w;
    const double t_mem = 40.0 * w / 6537e3, t_fir = fl / 36.4e6;  // us at the measured copy / DFMA peaks
    printf("q=%3d occ %d | tma full %7.1f  noFIR %7.1f  noState %7.1f  neither %7.1f us | "
           "roofline max(mem %.1f, fp64 %.1f) -> %.0f%%\n",
           q, o2, t_tma[0], t_tma[1], t_tma[2], t_tma[3], t_mem, t_fir, 100.0 * std::max(t_mem, t_fir) / t_tma[0]);
    {  // phase timestamps (one extra run)
      unsigned long long* st;
      CK(cudaMalloc(&st, sizeof(unsigned long long) * 8 * ntile));
      CK(cudaMemset(st, 0, sizeof(unsigned long long) * 8 * ntile));
      a.stamps = st;
      k_lsar_pass_tma<<<(unsigned)ntile, kPassThreads, sm2>>>(a);
      CK(cudaDeviceSynchronize());
      a.stamps = nullptr;
      std::vector<unsigned long long> hs(8 * ntile);
      CK(cudaMemcpy(hs.data(), st, sizeof(unsigned long long) * 8 * ntile, cudaMemcpyDeviceToHost));
      cudaFree(st);
      double acc[7] = {0};
      for (int64_t b = 0; b < ntile; ++b)
        for (int i = 1; i < 7; ++i) acc[i] += (double)(hs[8 * b + i] - hs[8 * b + i - 1]);
      printf("      phases (ns/CTA): issue+fill %.0f  ywait %.0f  fir %.0f  swait %.0f  update %.0f  partials %.0f\n",
             acc[1] / ntile, acc[2] / ntile, acc[3] / ntile, acc[4] / ntile, acc[5] / ntile, acc[6] / ntile);
    }
  }
  return 0;
}
