// Standalone check + timing of the INT8 tensor-core (Ozaki) Gram against the
// double-double CUDA-core Gram on correlated, weighted rows (AR(1) phi = 0.999
// windows, log-uniform weights): both produce (Gh, Gl); the difference is
// reported relative to sqrt(G_ii G_jj).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2112_12994_b200/csrc \
//        tools/i8gram_check.cu -o tools/bin/i8gram_check && tools/bin/i8gram_check [c K]
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include "k_gram.cuh"
#include "k_i8gram.cuh"
using namespace tfk;

#define CKE(x)                                                                      \
  do {                                                                              \
    cudaError_t e_ = (x);                                                           \
    if (e_ != cudaSuccess) {                                                        \
      fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
      exit(1);                                                                      \
    }                                                                               \
  } while (0)

int main(int argc, char** argv) {
  const int64_t c = argc > 1 ? atoll(argv[1]) : 200000;
  const int K = argc > 2 ? atoi(argv[2]) : 501;
  int sm = 0;
  CKE(cudaDeviceGetAttribute(&sm, cudaDevAttrMultiProcessorCount, 0));
  std::mt19937_64 g(7);
  std::normal_distribution<double> nd;
  std::uniform_real_distribution<double> ud(-2.0, 2.0);
  const int64_t n = c + K + 1000;
  std::vector<double> y(n);
  double v = 0.0;
  for (int64_t t = 0; t < n; ++t) y[t] = v = 0.999 * v + nd(g) * 1e3;
  std::vector<double> A((size_t)c * K);
  for (int64_t t = 0; t < c; ++t) {
    const int64_t s = (int64_t)(g() % (uint64_t)(n - K));
    const double w = std::pow(10.0, ud(g));
    for (int j = 0; j < K; ++j) A[(size_t)t * K + j] = w * y[s + j];
  }
  double* dA;
  CKE(cudaMalloc(&dA, A.size() * 8));
  CKE(cudaMemcpy(dA, A.data(), A.size() * 8, cudaMemcpyHostToDevice));
  DenseRows ld{dA, K};
  const int64_t KK = (int64_t)K * K;
  // ---- dd path
  const GramDDPlan gp = gram_dd_plan(c, K, sm);
  double *W, *cnp, *cn, *Gh, *Gl, *Ih, *Il;
  const unsigned ns = (unsigned)((c + kCnRows - 1) / kCnRows);
  CKE(cudaMalloc(&W, (size_t)gp.npair * gp.nsplit * 8192 * 8));
  CKE(cudaMalloc(&cnp, (size_t)ns * K * 8));
  CKE(cudaMalloc(&cn, K * 8));
  CKE(cudaMalloc(&Gh, KK * 8));
  CKE(cudaMalloc(&Gl, KK * 8));
  CKE(cudaMalloc(&Ih, KK * 8));
  CKE(cudaMalloc(&Il, KK * 8));
  auto run_dd = [&]() {
    k_colnorm2_part<DenseRows><<<dim3((K + 63) / 64, ns), 256>>>(ld, c, K, nullptr, cnp);
    k_colnorm2_sum<<<(K + 127) / 128, 128>>>(cnp, (int)ns, K, cn);
    k_gram_dd<DenseRows><<<dim3(gp.npair, gp.nsplit), kDDThreads>>>(ld, c, K, gp.nblk, gp.rps, gp.nsplit, W, nullptr, cn);
    k_gram_dd_reduce<<<(unsigned)(((int64_t)gp.npair * 4096 + 255) / 256), 256>>>(W, gp.npair, gp.nsplit, gp.nblk, K,
                                                                                  Gh, Gl, nullptr);
  };
  // ---- int8 path
  const int Kp = (K + kI8Tile - 1) / kI8Tile * kI8Tile;
  const int64_t cpad = (c + kI8Tile - 1) / kI8Tile * kI8Tile;
  const int nbs = Kp / kI8Tile, nbt = kI8S * nbs;
  std::vector<int2> tiles;
  std::vector<int> tile_of((size_t)nbt * nbt, -1);
  for (int I = 0; I < nbt; ++I)
    for (int J = I; J < nbt; ++J)
      if (I / nbs + J / nbs <= kI8S - 1) {
        tile_of[(size_t)I * nbt + J] = (int)tiles.size();
        tiles.push_back(make_int2(I, J));
      }
  printf("c %lld K %d: %zu int8 tiles of 128x128 (%d digit planes), dd plan %d pairs x %d splits\n", (long long)c, K,
         tiles.size(), kI8S, gp.npair, gp.nsplit);
  int8_t* D;
  int *E, *dtile_of;
  int2* dtiles;
  int32_t* P;
  double* mpart;
  CKE(cudaMalloc(&D, (size_t)kI8S * Kp * cpad));
  CKE(cudaMalloc(&E, Kp * 4));
  CKE(cudaMalloc(&mpart, (size_t)ns * K * 8));
  CKE(cudaMalloc(&dtiles, tiles.size() * sizeof(int2)));
  CKE(cudaMalloc(&dtile_of, tile_of.size() * 4));
  CKE(cudaMalloc(&P, tiles.size() * 128 * 128 * 4));
  CKE(cudaMemcpy(dtiles, tiles.data(), tiles.size() * sizeof(int2), cudaMemcpyHostToDevice));
  CKE(cudaMemcpy(dtile_of, tile_of.data(), tile_of.size() * 4, cudaMemcpyHostToDevice));
  CKE(cudaFuncSetAttribute(k_i8_gemm, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kI8Smem));
  cudaEvent_t ev[5];
  for (auto& e : ev) CKE(cudaEventCreate(&e));
  auto run_i8 = [&]() {
    cudaEventRecord(ev[0]);
    k_i8_colmax_part<DenseRows><<<dim3((K + 63) / 64, ns), 256>>>(ld, c, K, nullptr, mpart);
    k_i8_colmax_fin<<<(K + 127) / 128, 128>>>(mpart, (int)ns, K, E);
    k_i8_slice<DenseRows><<<dim3((unsigned)(cpad / kI8Tile), Kp / 32), 256>>>(ld, c, K, Kp, cpad / kI8Tile, nullptr, E, D);
    cudaEventRecord(ev[1]);
    k_i8_gemm<<<(unsigned)tiles.size(), kI8Threads, kI8Smem>>>(D, cpad / kI8Tile, dtiles, P);
    cudaEventRecord(ev[2]);
    k_i8_combine<<<(unsigned)((KK + 255) / 256), 256>>>(P, dtile_of, nbt, K, Kp, E, Ih, Il);
    cudaEventRecord(ev[3]);
  };
  run_dd();
  run_i8();
  CKE(cudaGetLastError());
  CKE(cudaDeviceSynchronize());
  std::vector<double> gh(KK), gl(KK), ih(KK), il(KK);
  CKE(cudaMemcpy(gh.data(), Gh, KK * 8, cudaMemcpyDeviceToHost));
  CKE(cudaMemcpy(gl.data(), Gl, KK * 8, cudaMemcpyDeviceToHost));
  CKE(cudaMemcpy(ih.data(), Ih, KK * 8, cudaMemcpyDeviceToHost));
  CKE(cudaMemcpy(il.data(), Il, KK * 8, cudaMemcpyDeviceToHost));
  double worst = 0.0, worst_hi = 0.0;
  int wi = 0, wj = 0;
  for (int i = 0; i < K; ++i)
    for (int j = 0; j < K; ++j) {
      const size_t e = (size_t)i * K + j;
      const double d = (gh[e] - ih[e]) + (gl[e] - il[e]);
      const double sc = std::sqrt(gh[(size_t)i * K + i] * gh[(size_t)j * K + j]);
      const double r = std::fabs(d) / sc;
      if (r > worst) worst = r, wi = i, wj = j;
      worst_hi = std::max(worst_hi, std::fabs(gh[e] - ih[e]) / sc);
    }
  printf("max |G_dd - G_i8| / sqrt(G_ii G_jj) = %.3e at (%d, %d)  [hi words: %.3e]\n", worst, wi, wj, worst_hi);
  // timing
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(a);
    run_dd();
    cudaEventRecord(b);
    CKE(cudaEventSynchronize(b));
    float tdd;
    cudaEventElapsedTime(&tdd, a, b);
    run_i8();
    CKE(cudaEventSynchronize(ev[3]));
    float t1, t2, t3;
    cudaEventElapsedTime(&t1, ev[0], ev[1]);
    cudaEventElapsedTime(&t2, ev[1], ev[2]);
    cudaEventElapsedTime(&t3, ev[2], ev[3]);
    const double ops = 2.0 * tiles.size() * 128.0 * 128.0 * cpad;
    const double l2b = (double)tiles.size() * 2 * 128 * cpad;
    printf("dd %.3f ms | i8: slice %.3f ms, gemm %.3f ms (%.0f TOPS, %.1f TB/s L2->smem), combine %.3f ms, total %.3f ms\n",
           tdd, t1, t2, ops / t2 / 1e9, l2b / t2 / 1e9, t3, t1 + t2 + t3);
  }
  CKE(cudaGetLastError());
  return worst < 1e-22 ? 0 : 2;
}
