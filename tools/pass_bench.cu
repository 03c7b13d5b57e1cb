// pass_bench.cu -- the fused LSAR pass kernels in isolation (development helper).
// Times k_lsar_pass_pst over w = 1e7 rows at several lags, also with its
// debug variants (template DBG bit 2: no FIR, bit 3: no state traffic) to split the
// cost into memory and FIR parts, and k_lsar_pass (exact tap order) at q < 16.
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
int main(int argc, char** argv) {
  const int only_q = argc > 1 ? atoi(argv[1]) : -1;  // profile mode: one launch of the pst kernel at this lag
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
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  if (only_q >= 0) {
    a.q = only_q;
    const size_t smp = PassLayout(only_q).bytes();
    CK(cudaFuncSetAttribute(k_lsar_pass_pst<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smp));
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_lsar_pass_pst<0>, kPassThreads, smp);
    const unsigned grid = (unsigned)std::min<int64_t>(ntile, (int64_t)occ * nsm);
    k_lsar_pass_pst<0><<<grid, kPassThreads, smp>>>(a);
    CK(cudaDeviceSynchronize());
    printf("one launch at q=%d done\n", only_q);
    return 0;
  }
  for (int q : {1, 8, 15, 16, 50, 100, 200, 500}) {
    a.q = q;
      const double fl = 2.0 * (q + 1) * w;
    const double t_mem = 40.0 * w / 6537e3, t_fir = fl / 36.4e6;  // us at the measured copy / DFMA peaks
    double t_core = 0;
    if (q < 16) {  // CUDA-core pass (exact tap order)
      const size_t sm0 = pass_smem_bytes(q);
      CK(cudaFuncSetAttribute(k_lsar_pass, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm0));
      t_core = timeit([&] { k_lsar_pass<<<(unsigned)ntile, kPassThreads, sm0>>>(a); });
    }
    const size_t smp = PassLayout(q).bytes();
    CK(cudaFuncSetAttribute(k_lsar_pass_pst<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smp));
    CK(cudaFuncSetAttribute(k_lsar_pass_pst<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smp));
    CK(cudaFuncSetAttribute(k_lsar_pass_pst<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smp));
    CK(cudaFuncSetAttribute(k_lsar_pass_pst<12>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smp));
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_lsar_pass_pst<0>, kPassThreads, smp);
    const unsigned grid = (unsigned)std::min<int64_t>(ntile, (int64_t)occ * nsm);
    double tp[4];
    tp[0] = timeit([&] { k_lsar_pass_pst<0><<<grid, kPassThreads, smp>>>(a); });
    tp[1] = timeit([&] { k_lsar_pass_pst<4><<<grid, kPassThreads, smp>>>(a); });
    tp[2] = timeit([&] { k_lsar_pass_pst<8><<<grid, kPassThreads, smp>>>(a); });
    tp[3] = timeit([&] { k_lsar_pass_pst<12><<<grid, kPassThreads, smp>>>(a); });
    CK(cudaGetLastError());
    printf("q=%3d pst occ %d | full %7.1f  noFIR %7.1f  noState %7.1f  neither %7.1f us | roofline max(mem %.1f, "
           "fp64 %.1f) -> %.0f%%",
           q, occ, tp[0], tp[1], tp[2], tp[3], t_mem, t_fir, 100.0 * std::max(t_mem, t_fir) / tp[0]);
    if (q < 16) printf(" | k_lsar_pass %.1f us", t_core);
    printf("\n");
    if (q < 16) {  // agreement with the exact-order kernel
      std::vector<double> s1(w), r1(w), s2(w), r2(w);
      const size_t sm0 = pass_smem_bytes(q);
      CK(cudaMemcpy(s, hy.data(), sizeof(double) * w, cudaMemcpyHostToDevice));
      CK(cudaMemcpy(r, hy.data() + 1, sizeof(double) * w, cudaMemcpyHostToDevice));
      k_lsar_pass<<<(unsigned)ntile, kPassThreads, sm0>>>(a);
      CK(cudaMemcpy(s1.data(), s, sizeof(double) * w, cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(r1.data(), r, sizeof(double) * w, cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(s, hy.data(), sizeof(double) * w, cudaMemcpyHostToDevice));
      CK(cudaMemcpy(r, hy.data() + 1, sizeof(double) * w, cudaMemcpyHostToDevice));
      k_lsar_pass_pst<0><<<grid, kPassThreads, smp>>>(a);
      CK(cudaMemcpy(s2.data(), s, sizeof(double) * w, cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(r2.data(), r, sizeof(double) * w, cudaMemcpyDeviceToHost));
      double ds = 0, dr = 0;
      for (int64_t i = 0; i < w; ++i) {
        ds = std::max(ds, std::abs(s1[i] - s2[i]) / std::max(std::abs(s1[i]), 1e-300));
        dr = std::max(dr, std::abs(r1[i] - r2[i]) / (std::abs(r1[i]) + 1e-3));
      }
      printf("      pst vs exact-order: s max rel %.2e, r max rel %.2e\n", ds, dr);
    }
  }
  return 0;
}
