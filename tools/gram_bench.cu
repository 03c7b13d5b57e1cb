// gram_bench.cu -- microbenchmark of the split-K DMMA Gram kernels on dense Q.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2112_12994_b200/csrc gram_bench.cu -o gram_bench
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "k_gram.cuh"

using namespace tfk;

#define CK(x)                                                                         \
  do {                                                                                \
    cudaError_t e = (x);                                                              \
    if (e != cudaSuccess) {                                                           \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      exit(1);                                                                        \
    }                                                                                 \
  } while (0)

struct Plan {
  int nblk, npair, nsplit;
  int64_t rps;
};
static Plan plan(int64_t rows, int K, int sms, int per_sm, int bw) {
  Plan g;
  g.nblk = (K + bw - 1) / bw;
  g.npair = g.nblk * (g.nblk + 1) / 2;
  const int64_t target = (int64_t)per_sm * sms;
  int64_t ns = (target + g.npair - 1) / g.npair;
  ns = std::max<int64_t>(1, std::min<int64_t>(ns, (rows + 255) / 256));
  int64_t rps = (rows + ns - 1) / ns;
  rps = (rps + 31) / 32 * 32;
  g.rps = std::max<int64_t>(rps, 32);
  g.nsplit = (int)((rows + g.rps - 1) / g.rps);
  return g;
}

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const int64_t cmax = 200000;
  const int Kmax = 512;
  double* Q;
  CK(cudaMalloc(&Q, sizeof(double) * cmax * (Kmax + 4)));
  std::vector<double> h((size_t)cmax * (Kmax + 4));
  for (size_t i = 0; i < h.size(); ++i) h[i] = std::sin(0.37 * (double)i) * 0.5;
  CK(cudaMemcpy(Q, h.data(), sizeof(double) * h.size(), cudaMemcpyHostToDevice));
  double *W, *G;
  int* tickets;
  CK(cudaMalloc(&W, sizeof(double) * 64 * 1024 * 1024));
  CK(cudaMalloc(&G, sizeof(double) * 1024 * 1024));
  CK(cudaMalloc(&tickets, sizeof(int) * 4096));
  CK(cudaMemset(tickets, 0, sizeof(int) * 4096));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  printf("%8s %5s %7s %7s %10s %9s\n", "c", "K", "nsplit", "npair", "us", "TF/s(alg)");
  for (int64_t c : {10000LL, 100000LL, 200000LL}) {
    for (int K : {64, 101, 151, 201, 301, 501}) {
      for (int variant = 0; variant < 5; ++variant) {
        static const int vst[5] = {2, 3, 4, 3, 2}, vslab[5] = {32, 16, 16, 32, 16};
        const int stages = vst[variant], slab = vslab[variant];
        Plan g = plan(c, K, sms, 4, 64);
        const int64_t ldq = (K + 1) / 2 * 2;
        dim3 grid(g.npair, g.nsplit);
        const size_t sm2 = gram2_smem_bytes(stages, slab);
        auto kern = [&]() -> void (*)(const double*, int64_t, int64_t, int, int, int64_t, double*, const int*) {
          switch (variant) {
            case 0: return k_gram_dense_t<2, 32>;
            case 1: return k_gram_dense_t<3, 16>;
            case 2: return k_gram_dense_t<4, 16>;
            case 3: return k_gram_dense_t<3, 32>;
            default: return k_gram_dense_t<2, 16>;
          }
        }();
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm2));
        int occ = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kGramThreads, sm2));
        auto run = [&]() {
          kern<<<grid, kGramThreads, sm2>>>(Q, ldq, c, K, g.nblk, g.rps, W, nullptr);
          k_gram_reduce<<<g.npair * 128, 256>>>(W, g.npair, g.nsplit, g.nblk, K, G, nullptr);
        };
        for (int it = 0; it < 3; ++it) run();
        CK(cudaEventRecord(e0));
        const int reps = 20;
        for (int it = 0; it < reps; ++it) run();
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        const double us = ms * 1e3 / reps;
        const double flop = (double)c * K * (K + 1);
        printf("%8lld %5d %7d %7d %10.1f %9.2f  (stages %d, slab %d, occ %d)\n", (long long)c, K, g.nsplit, g.npair, us,
               flop / (us * 1e-6) / 1e12, stages, slab, occ);
      }
    }
  }
  CK(cudaGetLastError());
  return 0;
}
