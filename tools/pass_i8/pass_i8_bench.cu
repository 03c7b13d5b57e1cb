// pass_i8_bench.cu -- the INT8 tensor-core sweep pass (k_lsar_pass_i8) against
// the fp64 DMMA pass (k_lsar_pass_pst) in isolation: w = 1e8 rows, several
// lags; residual agreement (relative to eps * sum |phi| |y|), then times of
// both and of the int8 kernel's debug variants (bit 0: no MMAs, bit 1: no
// epilogue arithmetic / traffic) to split MMA, epilogue and load costs.
// build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -I paper_2112_12994_b200/csrc \
//          -I tools/pass_i8 tools/pass_i8/pass_i8_bench.cu -o tools/bin/pass_i8_bench
#include <cuda_runtime.h>
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include "k_pass_i8.cuh"
using namespace tfk;
#define CK(x)                                                           \
  do {                                                                  \
    cudaError_t e = (x);                                                \
    if (e != cudaSuccess) {                                             \
      printf("CUDA %s line %d\n", cudaGetErrorString(e), __LINE__);     \
      exit(1);                                                          \
    }                                                                   \
  } while (0)

int main(int argc, char** argv) {
  const int64_t w = argc > 1 ? (int64_t)atof(argv[1]) : 100000000;
  const int64_t n = w + 700;
  std::vector<double> hy(n + 64, 0.0);
  std::mt19937_64 g(1);
  std::normal_distribution<double> nd;
  double v = 0.0;
  for (int64_t t = 0; t < n; ++t) hy[t] = v = 0.9 * v + nd(g) * 1e3;
  double m = 0.0;
  for (int64_t t = 0; t < n; ++t) m = std::max(m, std::fabs(hy[t]));
  int e = 0;
  std::frexp(m, &e);
  const int ey = e + 1;
  double *y, *s, *r, *s0, *r0, *cA, *cB, *tA, *tB, *phi, *R;
  CK(cudaMalloc(&y, sizeof(double) * hy.size()));
  CK(cudaMemcpy(y, hy.data(), sizeof(double) * hy.size(), cudaMemcpyHostToDevice));
  for (double** p : {&s, &r, &s0, &r0}) CK(cudaMalloc(p, sizeof(double) * w));
  CK(cudaMemcpy(s0, hy.data(), sizeof(double) * w, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(r0, hy.data() + 1, sizeof(double) * w, cudaMemcpyHostToDevice));
  CK(cudaMalloc(&cA, sizeof(double) * (w / 32 + 2)));
  CK(cudaMalloc(&cB, sizeof(double) * (w / 32 + 2)));
  const int64_t ntile = (w + kPassTile - 1) / kPassTile;
  CK(cudaMalloc(&tA, sizeof(double) * ntile));
  CK(cudaMalloc(&tB, sizeof(double) * ntile));
  std::vector<double> hp(1024);
  for (auto& x : hp) x = 0.02 * nd(g);
  CK(cudaMalloc(&phi, sizeof(double) * 1024));
  CK(cudaMemcpy(phi, hp.data(), sizeof(double) * 1024, cudaMemcpyHostToDevice));
  CK(cudaMalloc(&R, sizeof(double)));
  const double Rv = 1e6 * (double)w;
  CK(cudaMemcpy(R, &Rv, sizeof(double), cudaMemcpyHostToDevice));
  const int64_t stride = (n + kPiPlaneHalo + 255) / 256 * 256;
  int8_t* yp;
  int* dey;
  CK(cudaMalloc(&yp, (size_t)kPiSY * stride));
  CK(cudaMalloc(&dey, sizeof(int)));
  CK(cudaMemcpy(dey, &ey, sizeof(int), cudaMemcpyHostToDevice));
  k_y_planes<<<(unsigned)((stride / 16 + 255) / 256), 256>>>(y, n, stride, ey, stride, yp);
  CK(cudaDeviceSynchronize());
  PassArgs a{};
  a.y = y;
  a.w = w;
  a.phi = phi;
  a.s = s;
  a.r = r;
  a.Rprev = R;
  a.chunkA = cA;
  a.chunkB = cB;
  a.tileA = tA;
  a.tileB = tB;
  a.ylen = n + 64;
  PassI8Args ia{};
  ia.yp = yp;
  ia.yp_stride = stride;
  ia.ey = dey;
  int nsm = 0;
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto launch_pst = [&](int q) {
    a.q = q;
    const size_t smem = PassLayout(q).bytes();
    cudaFuncSetAttribute(k_lsar_pass_pst<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_lsar_pass_pst<0>, kPassThreads, smem);
    k_lsar_pass_pst<0><<<(unsigned)std::min<int64_t>(ntile, (int64_t)occ * nsm), kPassThreads, smem>>>(a);
  };
  auto launch_i8 = [&](int q, int dbg) {
    a.q = q;
    ia.a = a;
    const size_t smem = PassI8Layout(q).bytes;
    const unsigned grid = (unsigned)std::min<int64_t>(ntile, nsm);
    switch (dbg) {
      case 0:
        cudaFuncSetAttribute(k_lsar_pass_i8<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k_lsar_pass_i8<0><<<grid, kPiThreads, smem>>>(ia);
        break;
      case 1:
        cudaFuncSetAttribute(k_lsar_pass_i8<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k_lsar_pass_i8<1><<<grid, kPiThreads, smem>>>(ia);
        break;
      case 2:
        cudaFuncSetAttribute(k_lsar_pass_i8<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k_lsar_pass_i8<2><<<grid, kPiThreads, smem>>>(ia);
        break;
      default:
        cudaFuncSetAttribute(k_lsar_pass_i8<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k_lsar_pass_i8<3><<<grid, kPiThreads, smem>>>(ia);
        break;
    }
  };
  auto reset = [&]() {
    CK(cudaMemcpy(s, s0, sizeof(double) * w, cudaMemcpyDeviceToDevice));
    CK(cudaMemcpy(r, r0, sizeof(double) * w, cudaMemcpyDeviceToDevice));
  };
  auto timeit = [&](auto f) {
    for (int i = 0; i < 2; ++i) f();
    CK(cudaDeviceSynchronize());
    const int reps = 5;
    cudaEventRecord(e0);
    for (int i = 0; i < reps; ++i) f();
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    return ms / reps;
  };
  if (argc > 3) {  // profile mode: one launch of the int8 kernel (lag argv[2], debug bits argv[3])
    reset();
    launch_i8(atoi(argv[2]), atoi(argv[3]));
    CK(cudaDeviceSynchronize());
    return 0;
  }
  std::vector<double> r1(w), r2(w), s1(w), s2(w), c1(w / 32 + 1), c2(w / 32 + 1);
  const int qs[] = {1, 2, 3, 16, 64, 128, 256, 400, 500, 640};
  printf("w %lld rows, E_y %d\n", (long long)w, ey);
  for (int q : qs) {
    reset();
    launch_pst(q);
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(r1.data(), r, sizeof(double) * w, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(s1.data(), s, sizeof(double) * w, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(c1.data(), cB, sizeof(double) * (w / 32), cudaMemcpyDeviceToHost));
    reset();
    launch_i8(q, 0);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(r2.data(), r, sizeof(double) * w, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(s2.data(), s, sizeof(double) * w, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(c2.data(), cB, sizeof(double) * (w / 32), cudaMemcpyDeviceToHost));
    double worst = 0.0, sworst = 0.0, cworst = 0.0, aphi = 1.0;
    int64_t wi = 0;
    for (int j = 0; j < q; ++j) aphi += std::fabs(hp[j]);
    for (int64_t i = 0; i < w; i += 7) {
      double sc = std::fabs(hy[i + q]);
      for (int j = 0; j < q; j += 1) sc += std::fabs(hp[j] * hy[i + q - 1 - j]);
      const double er = std::fabs(r1[i] - r2[i]) / (sc * 1.1102230246251565e-16);
      if (er > worst) worst = er, wi = i;
      sworst = std::max(sworst, std::fabs(s1[i] - s2[i]) / std::fabs(s1[i]));
      if (i > 200000000) break;
    }
    for (int64_t c = 0; c < w / 32; ++c) cworst = std::max(cworst, std::fabs(c1[c] - c2[c]) / std::fabs(c1[c]));
    if (worst > 50) {  // exact reference in long double for the worst row
      long double ex = -(long double)hy[wi + q];
      for (int j = 0; j < q; ++j) ex += (long double)hp[j] * (long double)hy[wi + q - 1 - j];
      printf("  worst row %lld (tile %lld): dmma %.17g i8 %.17g exact %.17Lg\n", (long long)wi, (long long)(wi / 2048),
             r1[wi], r2[wi], ex);
    }
    const float tp = timeit([&] { launch_pst(q); });
    const float t0 = timeit([&] { launch_i8(q, 0); });
    const float t1 = timeit([&] { launch_i8(q, 1); });
    const float t2 = timeit([&] { launch_i8(q, 2); });
    const float t3 = timeit([&] { launch_i8(q, 3); });
    printf("q %3d: |r_i8 - r_dmma| <= %.2f eps sum|phi y|, s rel %.1e, chunk ||r||^2 rel %.1e | dmma %.3f ms, i8 %.3f ms "
           "(no MMA %.3f, no epilogue %.3f, loads only %.3f) -> %.2fx\n",
           q, worst, sworst, cworst, tp, t0, t1, t2, t3, tp / t0);
  }
  return 0;
}
