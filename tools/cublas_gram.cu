#include <cublas_v2.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>
int main() {
  cublasHandle_t h; cublasCreate(&h);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (long c : {10000L, 100000L, 200000L}) for (int K : {101, 201, 301, 501}) {
    double *A, *C; cudaMalloc(&A, sizeof(double) * c * K); cudaMalloc(&C, sizeof(double) * K * K);
    std::vector<double> hA(c * K); for (size_t i = 0; i < hA.size(); ++i) hA[i] = ((i * 2654435761u) % 1000) * 1e-3;
    cudaMemcpy(A, hA.data(), sizeof(double) * hA.size(), cudaMemcpyHostToDevice);
    double one = 1, zero = 0;
    // A stored row-major c x K == column-major K x c (lda = K): C = A_cm * A_cm^T  (syrk N)
    auto run = [&] { cublasDsyrk(h, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_N, K, c, &one, A, K, &zero, C, K); };
    auto rung = [&] { cublasDgemm(h, CUBLAS_OP_N, CUBLAS_OP_T, K, K, c, &one, A, K, A, K, &zero, C, K); };
    for (int v = 0; v < 2; ++v) {
      for (int i = 0; i < 3; ++i) v ? rung() : run();
      cudaDeviceSynchronize(); cudaEventRecord(e0);
      for (int i = 0; i < 20; ++i) v ? rung() : run();
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double us = ms * 1e3 / 20;
      printf("%s c=%ld K=%d: %.1f us  %.2f TF/s (alg c*K*(K+1))\n", v ? "dgemm" : "dsyrk", c, K, us, (double)c * K * (K + 1) / us / 1e6);
    }
    cudaFree(A); cudaFree(C);
  }
  return 0;
}
