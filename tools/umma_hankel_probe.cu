// umma_hankel_probe.cu -- tcgen05.mma kind::i8 with a Hankel A operand read
// straight from a linear byte array (K-major no-swizzle descriptor with
// LBO = 16 B, SBO = 128 B: row a of A is bytes [16 a, 16 a + K)), a B operand
// of several stacked planes (N = 16 per plane), chains accumulating into
// TMEM column windows offset by 16 s (a diagonal "plane-sum" accumulator),
// TMEM zeroed by tcgen05.st so every MMA accumulates.  Compares with a CPU
// product.
// build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a tools/umma_hankel_probe.cu -o tools/bin/umma_hankel_probe
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

constexpr int M = 128, SY = 3, SP = 3, KB = 160;  // y planes, phi planes, K bytes
constexpr int NB = 16 * SP;                         // B rows (all phi planes)
constexpr int YLEN = 16 * M + KB;
constexpr int NCOL = 16 * (SY + SP - 1);

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ int lay(int r, int kb) { return (r >> 3) * (KB / 16) * 128 + (kb >> 4) * 128 + (r & 7) * 16 + (kb & 15); }
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}

// Y: [SY][YLEN] bytes; B: [NB][KB]; D: [M][NCOL]
__global__ void k_probe(const int8_t* Y, const int8_t* B, int32_t* D) {
  __shared__ __align__(1024) int8_t sy[SY][YLEN + 16];
  __shared__ __align__(1024) int8_t sb[NB * KB];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int e = tid; e < SY * YLEN; e += blockDim.x) sy[e / YLEN][e % YLEN] = Y[e];
  for (int e = tid; e < NB * KB; e += blockDim.x) sb[lay(e / KB, e % KB)] = B[e];
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)), "r"(128));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(1));
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base;
  // zero the accumulator columns (each warp its 32 lanes)
  {
    const uint32_t z = 0;
    for (int c0 = 0; c0 < NCOL; c0 += 8)
      asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(
                       tmem + ((uint32_t)(32 * warp) << 16) + (uint32_t)c0), "r"(z));
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (tid == 0) {
    for (int s = 0; s < SY; ++s) {
      const int nu = SP;  // all phi planes here
      const int N = 16 * nu;
      const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
      for (int k = 0; k < KB / 32; ++k) {
        const uint64_t da = sdesc(smem_u32(&sy[s][0]) + 32 * k, 16, 128);
        const uint64_t db = sdesc(smem_u32(sb) + k * 2 * 128, 128, (KB / 16) * 128);
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem + 16 * s),
            "l"(da), "l"(db), "r"(idesc), "r"(1));
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
  }
  {
    uint32_t done = 0;
    while (!done)
      asm volatile("{\n\t.reg .pred P;\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n\tselp.b32 %0, 1, 0, P;\n\t}"
                   : "=r"(done) : "r"(smem_u32(&bar)), "r"(0));
  }
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  for (int c0 = 0; c0 < NCOL; c0 += 8) {
    uint32_t v[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(tmem + ((uint32_t)(32 * warp) << 16) + (uint32_t)c0));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int j = 0; j < 8; ++j) D[(32 * warp + lane) * NCOL + c0 + j] = (int32_t)v[j];
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(128));
}

int main() {
  std::vector<int8_t> Y(SY * YLEN), B(NB * KB);
  srand(3);
  for (auto& v : Y) v = (int8_t)(rand() % 129 - 64);
  for (auto& v : B) v = (int8_t)(rand() % 129 - 64);
  int8_t *dY, *dB;
  int32_t* dD;
  cudaMalloc(&dY, Y.size());
  cudaMalloc(&dB, B.size());
  cudaMalloc(&dD, M * NCOL * 4);
  cudaMemcpy(dY, Y.data(), Y.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice);
  cudaMemset(dD, 0xff, M * NCOL * 4);
  k_probe<<<1, 128>>>(dY, dB, dD);
  cudaError_t e = cudaDeviceSynchronize();
  printf("kernel: %s\n", cudaGetErrorString(e));
  std::vector<int32_t> D(M * NCOL);
  cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
  long bad = 0;
  for (int a = 0; a < M; ++a)
    for (int col = 0; col < NCOL; ++col) {
      // column col = 16 d + b accumulates planes (s, u) with s + u = d: sum_k Y_s[16 a + k] B[16 u + b][k]
      const int d = col / 16, b = col % 16;
      int32_t ref = 0;
      for (int s = 0; s < SY; ++s) {
        const int u = d - s;
        if (u < 0 || u >= SP) continue;
        for (int k = 0; k < KB; ++k) ref += (int32_t)Y[s * YLEN + 16 * a + k] * (int32_t)B[(16 * u + b) * KB + k];
      }
      if (ref != D[a * NCOL + col]) {
        if (bad < 5) printf("mismatch (a %d, col %d): gpu %d ref %d\n", a, col, D[a * NCOL + col], ref);
        ++bad;
      }
    }
  printf("mismatches: %ld of %d\n", bad, M * NCOL);
  return bad ? 1 : 0;
}
