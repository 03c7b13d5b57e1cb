// Standalone timing harness for k_cholinv (development tool).
#define CI_TIMING 1
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <cmath>
__device__ long long g_ci_clk[256];
#define CI_STAMP(k) do { if (threadIdx.x == 0) g_ci_clk[(k)] = clock64(); } while (0)
#include "../paper_2112_12994_b200/csrc/k_cholinv.cuh"
using namespace tfk;
int main(int argc, char** argv) {
  int K = argc > 1 ? atoi(argv[1]) : 201;
  std::vector<double> A((size_t)400 * K), G((size_t)K * K, 0.0);
  srand(1);
  for (auto& v : A) v = (rand() / (double)RAND_MAX) - 0.5;
  for (int i = 0; i < K; ++i) for (int j = 0; j < K; ++j) { double s = 0; for (int t = 0; t < 400; ++t) s += A[t*K+i]*A[t*K+j]; G[i*K+j] = s; }
  const int64_t tsz = tpu_size(K);
  std::vector<double> Gt(tsz, 0.0);
  for (int i = 0; i < K; ++i) for (int j = i; j < K; ++j) Gt[tpu_idx(K, i, j)] = G[i*K+j];
  double *dG, *dR, *scr; int *flags, *status;
  cudaMalloc(&dG, sizeof(double)*tsz); cudaMalloc(&dR, sizeof(double)*tsz); cudaMalloc(&scr, sizeof(double)*40000);
  cudaMalloc(&flags, 16); cudaMalloc(&status, 16); cudaMemset(flags, 0, 16); cudaMemset(status, 0, 16);
  cudaMemcpy(dG, Gt.data(), sizeof(double)*tsz, cudaMemcpyHostToDevice);
  CholinvArgs a; a.G = dG; a.K = K; a.pass = 0; a.nrows = 400; a.RD = dR; a.use_smem = cholinv_in_smem(K); a.flags = flags; a.gate = nullptr; a.status = status; a.lag = 1; a.force_b = 0; a.invert = argc > 2 ? atoi(argv[2]) : 0;
  size_t smem = a.use_smem ? cholinv_smem_bytes(K) : 0;
  cudaFuncSetAttribute(k_cholinv, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(e0);
    k_cholinv<<<1, kCholinvThreads, smem>>>(a);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    long long clk[256]; cudaMemcpyFromSymbol(clk, g_ci_clk, sizeof(clk));
    printf("K=%d rep %d: %.1f us  err=%s\n", K, rep, ms*1e3, cudaGetErrorString(cudaGetLastError()));
    if (rep == 4) { for (int k = 1; k < 64; ++k) if (clk[k]) printf("  stamp %2d: +%lld cycles\n", k, clk[k]-clk[0]); }
  }
  // check: off-diagonal R tiles and Dinv diagonal tiles reproduce G:
  //   reconstruct R (invert the diagonal tiles on the host), then R^T R vs G
  std::vector<double> Rt(tsz); cudaMemcpy(Rt.data(), dR, sizeof(double)*tsz, cudaMemcpyDeviceToHost);
  std::vector<double> R((size_t)K*K, 0.0);
  for (int i = 0; i < K; ++i) for (int j = i; j < K; ++j) if ((i >> 5) != (j >> 5)) R[i*K+j] = Rt[tpu_idx(K, i, j)];
  for (int J = 0; J < (K + 31) / 32; ++J) {
    int m = std::min(32, K - 32*J); std::vector<double> X(m*m), Rb(m*m, 0.0);
    for (int i = 0; i < m; ++i) for (int j = i; j < m; ++j) X[i*m+j] = Rt[tpu_idx(K, 32*J+i, 32*J+j)];
    for (int j = 0; j < m; ++j) { for (int i = j; i >= 0; --i) { double s = (i==j) ? 1.0 : 0.0; for (int q = i+1; q <= j; ++q) s -= X[i*m+q]*Rb[q*m+j]; Rb[i*m+j] = s / X[i*m+i]; } }
    for (int i = 0; i < m; ++i) for (int j = i; j < m; ++j) R[(32*J+i)*K + 32*J+j] = Rb[i*m+j];
  }
  double maxerr = 0, gmax = 0;
  for (int i = 0; i < K; ++i) for (int j = i; j < K; ++j) { double s = 0; for (int q = 0; q <= i; ++q) s += R[q*K+i]*R[q*K+j]; maxerr = fmax(maxerr, fabs(s - G[i*K+j])); gmax = fmax(gmax, fabs(G[i*K+j])); }
  printf("R^T R vs G rel err %.3e\n", maxerr / gmax);
  return 0;
}
