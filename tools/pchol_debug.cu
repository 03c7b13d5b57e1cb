// Standalone check of k_pchol_dd + k_svd_minnorm on a dumped exact Gram
// (tools/pchol_case.bin: K, c, Gh[K][K], Gl[K][K], expected phi[p], rank).
#include <cstdio>
#include <vector>
#include <cmath>
#include "../paper_2112_12994_b200/csrc/k_exact.cuh"
using namespace tfk;
int main() {
  FILE* f = fopen("tools/pchol_case.bin", "rb");
  long long K, c; if (fread(&K, 8, 1, f) != 1 || fread(&c, 8, 1, f) != 1) return 1;
  const int p = (int)K - 1;
  std::vector<double> Gh(K * K), Gl(K * K), want(p); long long rank;
  if (fread(Gh.data(), 8, K * K, f) != (size_t)(K * K) || fread(Gl.data(), 8, K * K, f) != (size_t)(K * K) ||
      fread(want.data(), 8, p, f) != (size_t)p || fread(&rank, 8, 1, f) != 1) return 1;
  fclose(f);
  double *dGh, *dGl, *dRh, *dRl, *dN, *dsig, *dx, *dtol, *dphi; int *dperm, *dsvd, *dmeth, *drank;
  cudaMalloc(&dGh, K * K * 8); cudaMalloc(&dGl, K * K * 8); cudaMalloc(&dRh, K * K * 8); cudaMalloc(&dRl, K * K * 8);
  cudaMalloc(&dN, K * K * 8); cudaMalloc(&dsig, K * 8); cudaMalloc(&dx, 32 * K * 8); cudaMalloc(&dtol, 16);
  cudaMalloc(&dphi, K * 8); cudaMalloc(&dperm, K * 4); cudaMalloc(&dsvd, 80 * 4); cudaMalloc(&dmeth, 4); cudaMalloc(&drank, 4);
  cudaMemcpy(dGh, Gh.data(), K * K * 8, cudaMemcpyHostToDevice); cudaMemcpy(dGl, Gl.data(), K * K * 8, cudaMemcpyHostToDevice);
  ExactOut o{dphi, nullptr, 0, nullptr, dmeth, drank, 1};
  PcholArgs pa{}; pa.Gh = dGh; pa.Gl = dGl; pa.K = K; pa.rev = 0; pa.rows = c; pa.Rh = dRh; pa.Rl = dRl; pa.N = dN;
  pa.perm = dperm; pa.svd = dsvd; pa.tol = dtol; pa.o = o;
  double* dD; cudaMalloc(&dD, 4 * K * 8); pa.Dh = dD; pa.Dl = dD + 2 * K;
  { int pc = pchol_ctas(K); cudaLaunchConfig_t c0{}; c0.gridDim = dim3(pc); c0.blockDim = dim3(kPcThreads);
    cudaLaunchAttribute a0[1]; a0[0].id = cudaLaunchAttributeClusterDimension; a0[0].val.clusterDim.x = pc;
    a0[0].val.clusterDim.y = 1; a0[0].val.clusterDim.z = 1; c0.attrs = a0; c0.numAttrs = 1;
    cudaLaunchKernelEx(&c0, k_pchol_dd, pa); }
  int nct = std::min(16, std::max(1, (p + 31) / 32)), nblk = 2 * nct, bw = std::max(1, (p + nblk - 1) / nblk);
  SvdArgs a{}; a.N = dN; a.sig = dsig; a.xpart = dx; a.perm = dperm; a.svd = dsvd; a.tol = dtol; a.p = p; a.nblk = nblk;
  a.bw = bw; a.rev = 0; a.o = o;
  size_t smem = svd_smem_bytes(p, bw);
  cudaFuncSetAttribute((const void*)k_svd_minnorm, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncSetAttribute((const void*)k_svd_minnorm, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaLaunchConfig_t cfg{}; cfg.gridDim = dim3(nct); cfg.blockDim = dim3(kSvdThreads); cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = nct;
  at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1; cfg.attrs = at; cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, k_svd_minnorm, a);
  cudaError_t e2 = cudaDeviceSynchronize();
  std::vector<double> phi(p); int meth, rk; std::vector<int> sv(80);
  cudaMemcpy(phi.data(), dphi, p * 8, cudaMemcpyDeviceToHost); cudaMemcpy(&meth, dmeth, 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(&rk, drank, 4, cudaMemcpyDeviceToHost); cudaMemcpy(sv.data(), dsvd, 320, cudaMemcpyDeviceToHost);
  double err = 0, mx = 0;
  for (int i = 0; i < p; ++i) { err = fmax(err, fabs(phi[i] - want[i])); mx = fmax(mx, fabs(want[i])); }
  printf("pchol+svd: %s/%s method %d rank %d (want %lld) svdflag %d rel err %.3e phi0 %g want %g\n",
         cudaGetErrorString(e), cudaGetErrorString(e2), meth, rk, rank, sv[0], err / mx, phi[0], want[0]);
  std::vector<int> perm(K); std::vector<double> Rh(K * K), N(K * K);
  cudaMemcpy(perm.data(), dperm, K * 4, cudaMemcpyDeviceToHost); cudaMemcpy(Rh.data(), dRh, K * K * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(N.data(), dN, (size_t)p * (p + 1) * 8, cudaMemcpyDeviceToHost);
  const double mx0 = fabs(Rh[(size_t)perm[0] * K]);
  printf("perm:"); for (int k = 0; k < K; ++k) printf(" %d", perm[k]); printf("\nrkk/max:");
  for (int k = 0; k < p; ++k) printf(" %.3e", fabs(Rh[(size_t)perm[k] * K + k]) / mx0);
  printf("\nz:"); for (int k = 0; k < p; ++k) printf(" %.3e", Rh[(size_t)p * K + k]);
  printf("\nN col0:"); for (int j = 0; j <= p; ++j) printf(" %.3e", N[j]);
  printf("\n");
  return 0;
}
