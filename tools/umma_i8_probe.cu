// umma_i8_probe.cu -- minimal tcgen05.mma kind::i8 check (one CTA, 128 x 128
// int32 tile, K = 256 int8): smem K-major "interleave" layout, instruction
// descriptor, TMEM alloc / commit / ld.  Compares with a CPU product.
// build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a tools/umma_i8_probe.cu -o tools/bin/umma_i8_probe
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

constexpr int M = 128, N = 128, KB = 128;  // K in bytes (int8 elements)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// K-major interleave layout, 16-byte units: (r/8)*SBO + (k/16)*LBO + (r%8)
__device__ __forceinline__ int lay(int r, int kb) { return (r >> 3) * (KB / 16) * 128 + (kb >> 4) * 128 + (r & 7) * 16 + (kb & 15); }

__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version (sm100)
  // base_offset 0, lbo_mode 0, layout type 0 (SWIZZLE_NONE)
  return d;
}

__global__ void k_probe(const int8_t* A, const int8_t* B, int32_t* D, int* flag) {
  __shared__ __align__(1024) int8_t sa[M * KB];
  __shared__ __align__(1024) int8_t sb[N * KB];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int e = tid; e < M * KB; e += blockDim.x) {
    const int r = e / KB, kb = e % KB;
    sa[lay(r, kb)] = A[e];
    sb[lay(r, kb)] = B[e];
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)), "r"(128));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(1));
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base;
  // instruction descriptor: c s32 (2) bits 4-5, a s8 (1) bits 7-9, b s8 (1) bits 10-12, K-major,
  // n_dim = N >> 3 at bits 17-22, m_dim = M >> 4 at bits 24-28
  const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
  if (tid == 0) {
    for (int k = 0; k < KB / 32; ++k) {
      const uint64_t da = sdesc(smem_u32(sa) + k * 2 * 128, 128, (KB / 16) * 128);
      const uint64_t db = sdesc(smem_u32(sb) + k * 2 * 128, 128, (KB / 16) * 128);
      const uint32_t acc = k > 0 ? 1u : 0u;
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
          "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
          "l"(da), "l"(db), "r"(idesc), "r"(acc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
  }
  // wait for the MMAs
  {
    uint32_t done = 0;
    while (!done) {
      asm volatile("{\n\t.reg .pred P;\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n\tselp.b32 %0, 1, 0, P;\n\t}"
                   : "=r"(done) : "r"(smem_u32(&bar)), "r"(0));
    }
  }
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  // epilogue: warp w reads lanes 32w..32w+31, 8 columns at a time
  for (int c0 = 0; c0 < N; c0 += 8) {
    uint32_t v[8];
    const uint32_t taddr = tmem + ((uint32_t)(32 * warp) << 16) + (uint32_t)c0;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int j = 0; j < 8; ++j) D[(32 * warp + lane) * N + c0 + j] = (int32_t)v[j];
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(128));
  if (tid == 0) *flag = 1;
}

int main() {
  std::vector<int8_t> A(M * KB), B(N * KB);
  srand(1);
  for (auto& v : A) v = (int8_t)(rand() % 255 - 127);
  for (auto& v : B) v = (int8_t)(rand() % 255 - 127);
  int8_t *dA, *dB;
  int32_t* dD;
  int* dflag;
  cudaMalloc(&dA, A.size());
  cudaMalloc(&dB, B.size());
  cudaMalloc(&dD, M * N * 4);
  cudaMalloc(&dflag, 4);
  cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice);
  cudaMemset(dD, 0, M * N * 4);
  cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 0);
  k_probe<<<1, 128>>>(dA, dB, dD, dflag);
  cudaError_t e = cudaDeviceSynchronize();
  printf("kernel: %s\n", cudaGetErrorString(e));
  std::vector<int32_t> D(M * N);
  cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
  long bad = 0;
  for (int i = 0; i < M; ++i)
    for (int j = 0; j < N; ++j) {
      int32_t ref = 0;
      for (int k = 0; k < KB; ++k) ref += (int32_t)A[i * KB + k] * (int32_t)B[j * KB + k];
      if (ref != D[i * N + j]) {
        if (bad < 5) printf("mismatch (%d,%d): gpu %d ref %d\n", i, j, D[i * N + j], ref);
        ++bad;
      }
    }
  printf("mismatches: %ld of %d\n", bad, M * N);
  return 0;
}
