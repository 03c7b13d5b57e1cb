// Standalone check of k_svd_minnorm on a dumped case (tools/svd_case.bin:
// p, tol, perm[p+1], N[p][p+1] column-major, expected phi[p]).
#include <cstdio>
#include <vector>
#include <cmath>
#include "../paper_2112_12994_b200/csrc/k_exact.cuh"
using namespace tfk;
int main() {
  FILE* f = fopen("tools/svd_case.bin", "rb");
  long long p; double tol; fread(&p, 8, 1, f); fread(&tol, 8, 1, f);
  std::vector<int> perm(p + 1); fread(perm.data(), 4, p + 1, f);
  std::vector<double> N(p * (p + 1)), want(p); fread(N.data(), 8, N.size(), f); fread(want.data(), 8, p, f);
  fclose(f);
  double *dN, *dsig, *dx, *dtol, *dphi; int *dperm, *dsvd;
  cudaMalloc(&dN, N.size() * 8); cudaMalloc(&dsig, p * 8); cudaMalloc(&dx, 32 * p * 8); cudaMalloc(&dtol, 8);
  cudaMalloc(&dphi, p * 8); cudaMalloc(&dperm, (p + 1) * 4); cudaMalloc(&dsvd, 80 * 4);
  cudaMemcpy(dN, N.data(), N.size() * 8, cudaMemcpyHostToDevice); cudaMemcpy(dtol, &tol, 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dperm, perm.data(), (p + 1) * 4, cudaMemcpyHostToDevice);
  std::vector<int> sv(80, 0); sv[0] = 1; sv[66] = (int)p; cudaMemcpy(dsvd, sv.data(), 320, cudaMemcpyHostToDevice);
  int nct = std::min(16, std::max(1, (int)(p + 31) / 32)), nblk = 2 * nct, bw = std::max(1, (int)(p + nblk - 1) / nblk);
  SvdArgs a{}; a.N = dN; a.sig = dsig; a.xpart = dx; a.perm = dperm; a.svd = dsvd; a.tol = dtol; a.p = p; a.nblk = nblk;
  a.bw = bw; a.rev = 0; a.o.phi = dphi; a.o.lag = 1;
  size_t smem = svd_smem_bytes(p, bw);
  cudaFuncSetAttribute((const void*)k_svd_minnorm, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncSetAttribute((const void*)k_svd_minnorm, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaLaunchConfig_t cfg{}; cfg.gridDim = dim3(nct); cfg.blockDim = dim3(kSvdThreads); cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = nct;
  at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1; cfg.attrs = at; cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, k_svd_minnorm, a);
  cudaError_t e2 = cudaDeviceSynchronize();
  printf("launch %s / %s  nct %d bw %d smem %zu\n", cudaGetErrorString(e), cudaGetErrorString(e2), nct, bw, smem);
  std::vector<double> phi(p), sig(p); cudaMemcpy(phi.data(), dphi, p * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(sig.data(), dsig, p * 8, cudaMemcpyDeviceToHost); cudaMemcpy(sv.data(), dsvd, 320, cudaMemcpyDeviceToHost);
  double err = 0, mx = 0;
  for (int i = 0; i < p; ++i) { err = fmax(err, fabs(phi[i] - want[i])); mx = fmax(mx, fabs(want[i])); }
  int sweeps = 0; while (sweeps < 60 && sv[2 + sweeps]) ++sweeps;
  printf("phi[0..3] %g %g %g %g want %g %g %g %g  rel err %.3e sweeps %d sig0 %g\n", phi[0], phi[1], phi[2], phi[3],
         want[0], want[1], want[2], want[3], err / mx, sweeps + 1, sig[0]);
  return 0;
}
