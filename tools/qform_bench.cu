// qform_bench.cu -- Q1 = A T microbenchmark (gathered window rows, TPU upper T).
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <random>
#include <algorithm>
#include "k_gram.cuh"
using namespace tfk;
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s line %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)
int main() {
  const int64_t n = 10000000;
  std::vector<double> hy(n + 64);
  std::mt19937_64 g(1);
  std::normal_distribution<double> nd;
  for (auto& v : hy) v = nd(g);
  double *y, *wt, *T, *Q;
  int64_t* idx;
  CK(cudaMalloc(&y, sizeof(double) * hy.size()));
  CK(cudaMemcpy(y, hy.data(), sizeof(double) * hy.size(), cudaMemcpyHostToDevice));
  const int64_t cmax = 100000;
  std::vector<int64_t> hi(cmax);
  std::vector<double> hw(cmax);
  std::uniform_int_distribution<int64_t> ui(0, n - 600);
  for (int64_t t = 0; t < cmax; ++t) { hi[t] = ui(g); hw[t] = 1.0 + 0.001 * (t % 7); }
  std::sort(hi.begin(), hi.end());
  CK(cudaMalloc(&idx, sizeof(int64_t) * cmax));
  CK(cudaMalloc(&wt, sizeof(double) * cmax));
  CK(cudaMemcpy(idx, hi.data(), sizeof(int64_t) * cmax, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(wt, hw.data(), sizeof(double) * cmax, cudaMemcpyHostToDevice));
  CK(cudaMalloc(&T, sizeof(double) * 300000));
  std::vector<double> hT(300000);
  for (auto& v : hT) v = nd(g) * 0.1;
  CK(cudaMemcpy(T, hT.data(), sizeof(double) * hT.size(), cudaMemcpyHostToDevice));
  CK(cudaMalloc(&Q, sizeof(double) * cmax * 512));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int64_t c : {10000LL, 100000LL}) {
    for (int K : {65, 129, 201}) {
      const int64_t ldq = (K + 1) & ~1;
      dim3 grid((unsigned)((c + 63) / 64), (unsigned)((K + 63) / 64));
      WinFwd wf{y, idx, wt, 0};
      auto timeit = [&](auto launch, const char* name) {
        for (int i = 0; i < 3; ++i) launch();
        cudaEventRecord(e0);
        for (int i = 0; i < 20; ++i) launch();
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        const double us = ms * 1e3 / 20;
        double fma = 0;  // padded tile work
        for (int L0 = 0; L0 < K; L0 += 64) fma += 64.0 * std::min(K, L0 + 64);
        fma *= c;
        printf("c=%6lld K=%3d %-14s %8.1f us  %6.2f TFLOP/s (padded)\n", (long long)c, K, name, us, 2 * fma / (us * 1e-6) / 1e12);
      };
      {
        static bool once = false;
        if (!once) {
          cudaFuncSetAttribute(k_qform_pipe<WinFwd, 3, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)qform_pipe_smem<3>());
          cudaFuncSetAttribute(k_qform_pipe<WinFwd, 2, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)qform_pipe_smem<2>());
          cudaFuncSetAttribute(k_qform_pipe<WinDense, 3, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)qform_pipe_smem<3>());
          cudaFuncSetAttribute(k_qform_pipe<WinDense, 2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)qform_pipe_smem<2>());
          once = true;
        }
      }
      timeit([&] { k_qform_pipe<WinFwd, 3, false><<<grid, kGramThreads, qform_pipe_smem<3>()>>>(wf, c, K, T, Q, ldq, nullptr); }, "pipe3 gather");
      timeit([&] { k_qform_pipe<WinFwd, 2, false><<<grid, kGramThreads, qform_pipe_smem<2>()>>>(wf, c, K, T, Q, ldq, nullptr); }, "pipe2 gather");
      double* A = Q + cmax * 256;  // scratch
      WinDense wd{A, ldq};
      timeit([&] {
        k_gather_rows<WinFwd><<<(unsigned)((c + 7) / 8), dim3(32, 8)>>>(wf, c, K, A, ldq);
        k_qform_pipe<WinDense, 3, true><<<grid, kGramThreads, qform_pipe_smem<3>()>>>(wd, c, K, T, Q, ldq, nullptr);
      }, "gather+pipe3d");
      timeit([&] {
        k_gather_rows<WinFwd><<<(unsigned)((c + 7) / 8), dim3(32, 8)>>>(wf, c, K, A, ldq);
        k_qform_pipe<WinDense, 2, true><<<grid, kGramThreads, qform_pipe_smem<2>()>>>(wd, c, K, T, Q, ldq, nullptr);
      }, "gather+pipe2d");
      timeit([&] { k_gather_rows<WinFwd><<<(unsigned)((c + 7) / 8), dim3(32, 8)>>>(wf, c, K, A, ldq); }, "gather only");
      CK(cudaGetLastError());
    }
  }
  return 0;
}
