// k_gram.cuh -- fp64 tensor-core (DMMA m8n8k4) Gram and Q-formation kernels
// for the CholeskyQR2 solve of the sampled least-squares system
// (replaces the Eigen ColPivHouseholderQR call of toeplitz.cpp:57-71, fed by
// apply_sample, sketch.cpp:61-79).
//
// The sampled, weighted rows are never materialised as a separate matrix:
// row t of the augmented system in forward column order (k_tpu.cuh) is
//   a_t[a] = w_t * y[off + i_t + a],  a = 0..K-1   (K = p + 1, target last)
// a contiguous slice of the series -- the gather is fused into the tile
// loads (apply_sample's product w * y is formed exactly as the reference).
//
//   k_gram_dense_t + k_gram_reduce : split-K Gram of a dense tall matrix
//              (64x64 upper block pairs, cp.async ring, split partials summed
//              in split order -- deterministic).
//   k_qform_pipe : Q = A * B for an upper-triangular TPU right factor B
//              (the preconditioned Q1 = A T and CholeskyQR's Q = A R^-1), A
//              read as window rows of the series or as a dense matrix.
#pragma once

#include "common.cuh"
#include "k_tpu.cuh"

namespace tfk {

struct DenseRows {
  const double* q;
  int64_t ld;
  __device__ __forceinline__ double operator()(int64_t t, int col) const {
    return q[t * ld + col];
  }
  __device__ __forceinline__ const double* row(int64_t t) const { return q + t * ld; }
};

constexpr int kGramThreads = 128;
constexpr int kSJ = 68;  // padded row stride (doubles): conflict-free fragment loads

__device__ __forceinline__ void pair_from_index(int pair, int nblk, int& jb, int& lb) {
  int rem = pair;
  jb = 0;
  while (rem >= nblk - jb) {
    rem -= nblk - jb;
    ++jb;
  }
  lb = jb + rem;
}

// ---------------------------------------------------------------------------
// Dense Gram, pipelined: G = Q^T Q for a dense row-major Q (ld even, so rows
// are 16-byte aligned).  Each CTA owns one 64 x 64 upper tile pair and a
// contiguous row range; 32-row slabs of the two 64-column blocks stream into
// shared memory with cp.async (LDGSTS, 16 B, zero-fill past the last row) in
// a 2-stage ring (3 CTAs per SM; 2 stages beat 3 by 2-7 % in
// tools/gram_bench.cu), so global latency overlaps the DMMA work.
// Partial tiles go to W[split][pair][64 x 64]; k_gram_reduce sums them in
// split order (deterministic) with many CTAs.
constexpr int kG2Stages = 2;
constexpr int kG2Ld = 68;  // padded smem row (doubles): 544 B, 16-byte aligned, conflict-free fragments

__host__ __device__ inline size_t gram2_smem_bytes(int stages = kG2Stages, int slab = 32) {
  return (size_t)stages * 2 * slab * kG2Ld * sizeof(double);
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int src_bytes) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(gmem), "r"(src_bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

template <int ST, int SLAB = 32>
__global__ void __launch_bounds__(kGramThreads)
    k_gram_dense_t(const double* __restrict__ Q, int64_t ld, int64_t rows, int K, int nblk,
                 int64_t rows_per_split, double* __restrict__ W, const int* skip_flag) {
  if (skip_flag && *skip_flag == 0) return;
  extern __shared__ __align__(16) double g2s[];
  int jb, lb;
  pair_from_index(blockIdx.x, nblk, jb, lb);
  const bool diag = jb == lb;
  const int J0 = jb * 64, L0 = lb * 64;
  const int64_t rb = (int64_t)blockIdx.y * rows_per_split;
  const int64_t re = min(rows, rb + rows_per_split);
  const int nslab = (int)((re - rb + SLAB - 1) / SLAB);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp & 1, wn = warp >> 1;
  // 16-byte chunk assignment: SLAB rows x 32 chunks per operand, SLAB / 4 per thread
  auto issue = [&](int slab) {
    double* sj = g2s + (size_t)(slab % ST) * 2 * SLAB * kG2Ld;
    double* sl = sj + SLAB * kG2Ld;
    const int64_t r0 = rb + (int64_t)slab * SLAB;
#pragma unroll
    for (int u = 0; u < SLAB / 4; ++u) {
      const int ch = tid + kGramThreads * u;  // 0..1023
      const int rr = ch >> 5, cc = (ch & 31) * 2;
      const int64_t row = r0 + rr;
      const bool rok = row < re;
      {
        const int col = J0 + cc;
        const int nb = (rok && col < K) ? 16 : 0;
        cp_async16(sj + rr * kG2Ld + cc, Q + (nb ? row * ld + col : 0), nb);
      }
      if (!diag) {
        const int col = L0 + cc;
        const int nb = (rok && col < K) ? 16 : 0;
        cp_async16(sl + rr * kG2Ld + cc, Q + (nb ? row * ld + col : 0), nb);
      }
    }
  };
  // warp-uniform work trimming: 8-wide fragments past column K, and the strictly
  // lower 32 x 32 quadrant of a diagonal pair, are never multiplied (their
  // outputs are not stored)
  const int ni = min(4, max(0, (K - (J0 + 32 * wm) + 7) / 8));
  const int nj = min(4, max(0, (K - (L0 + 32 * wn) + 7) / 8));
  const bool wskip = (diag && wm > wn) || ni == 0 || nj == 0;
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
#pragma unroll
  for (int s = 0; s < ST - 1; ++s) {
    if (s < nslab) issue(s);
    cp_async_commit();
  }
  for (int s = 0; s < nslab; ++s) {
    cp_async_wait<ST - 2>();
    __syncthreads();
    // refill the stage consumed in the previous iteration
    if (s + ST - 1 < nslab) issue(s + ST - 1);
    cp_async_commit();
    const double* SJ = g2s + (size_t)(s % ST) * 2 * SLAB * kG2Ld;
    const double* SL = diag ? SJ : SJ + SLAB * kG2Ld;
    // full 32 x 32 warp tiles take an unpredicated path: a predicated
    // mma.sync costs a WARPSYNC + NOP + ISETP per DMMA
    auto ksteps = [&](auto full) {
#pragma unroll
      for (int kk = 0; kk < SLAB / 4; ++kk) {
        const int tr = 4 * kk + (lane & 3);
        double af[4], bf[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) af[i] = SJ[tr * kG2Ld + 32 * wm + 8 * i + (lane >> 2)];
#pragma unroll
        for (int j = 0; j < 4; ++j) bf[j] = SL[tr * kG2Ld + 32 * wn + 8 * j + (lane >> 2)];
        dmma_4x4<decltype(full)::value>(acc, af, bf, ni, nj);
      }
    };
    if (!wskip) {
      if (ni == 4 && nj == 4) ksteps(std::true_type{});
      else ksteps(std::false_type{});
    }
  }
  cp_async_wait<0>();
  double* out = W + ((size_t)blockIdx.y * gridDim.x + blockIdx.x) * 4096;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int row = 32 * wm + 8 * i + (lane >> 2);
      const int col = 32 * wn + 8 * j + 2 * (lane & 3);
      *reinterpret_cast<double2*>(out + row * 64 + col) = make_double2(acc[i][j][0], acc[i][j][1]);
    }
}

// dense copy of loader rows (row-major, leading dimension ld >= K, even)
template <class L>
__global__ void k_rows_dense(L ld, int64_t rows, int K, double* __restrict__ out, int64_t ldo) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.y + threadIdx.y;
  if (t >= rows) return;
  for (int j = threadIdx.x; j < K; j += blockDim.x) out[t * ldo + j] = ld(t, j);
}

// G (TPU) = sum over splits of W[split][pair] in split order.  Block: 8 warps,
// 32 consecutive tile elements of one pair; warp w sums splits w, w + 8, ...;
// the 8 warp partials are then added in warp order.
__global__ void __launch_bounds__(256)
    k_gram_reduce(const double* __restrict__ W, int npair, int nsplit, int nblk, int K,
                  double* __restrict__ G, const int* skip_flag) {
  if (skip_flag && *skip_flag == 0) return;
  __shared__ double part[8][33];
  const int pair = blockIdx.x / 128, grp = blockIdx.x % 128;
  int jb, lb;
  pair_from_index(pair, nblk, jb, lb);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int e = grp * 32 + lane;          // element of the 64 x 64 tile (row-major)
  const int row = jb * 64 + (e >> 6), col = lb * 64 + (e & 63);
  const bool rowok = jb * 64 + ((grp * 32) >> 6) < K;  // whole group shares one tile row
  if (!rowok) return;
  const size_t sstride = (size_t)npair * 4096;
  const double* wp = W + (size_t)pair * 4096 + e;
  double s0 = 0.0, s1 = 0.0;
  int sp = warp;
  for (; sp + 8 < nsplit; sp += 16) {
    s0 += __ldcg(wp + (size_t)sp * sstride);
    s1 += __ldcg(wp + (size_t)(sp + 8) * sstride);
  }
  if (sp < nsplit) s0 += __ldcg(wp + (size_t)sp * sstride);
  part[warp][lane] = s0 + s1;
  __syncthreads();
  if (warp == 0) {
    double t = part[0][lane];
#pragma unroll
    for (int w = 1; w < 8; ++w) t += part[w][lane];
    if (row < K && col < K && (row <= col || (row >> 5) == (col >> 5))) G[tpu_idx(K, row, col)] = t;
  }
}

constexpr int kQA = 36;

// ---------------------------------------------------------------------------
// Window-row operands for k_qform_pipe: A(t, k) = weight(t) * row(t)[dir * k].
// The row pointers and weights of a CTA's 64 rows are read once into shared
// memory, so each 32-column chunk costs one global load per element (not the
// idx -> y dependent pair), and the weights scale the accumulator rows at the
// end instead of every loaded element.
struct WinFwd {  // w_t y[off + idx_t + k]
  const double* y;
  const int64_t* idx;
  const double* wt;
  int64_t off;
  __device__ __forceinline__ const double* row(int64_t t) const { return y + off + idx[t]; }
  static constexpr int dir = 1;
  __device__ __forceinline__ double weight(int64_t t) const { return wt[t]; }
};
struct WinRev {  // w_t y[base + idx_t - k]
  const double* y;
  const int64_t* idx;
  const double* wt;
  int64_t base;
  __device__ __forceinline__ const double* row(int64_t t) const { return y + base + idx[t]; }
  static constexpr int dir = -1;
  __device__ __forceinline__ double weight(int64_t t) const { return wt[t]; }
};
struct WinDense {  // q[t * ld + k]
  const double* q;
  int64_t ld;
  __device__ __forceinline__ const double* row(int64_t t) const { return q + t * ld; }
  static constexpr int dir = 1;
  __device__ __forceinline__ double weight(int64_t) const { return 1.0; }
};

// ---------------------------------------------------------------------------
// Pipelined window-row Q = A B: A chunks gathered with 8-byte cp.async (or
// 16-byte when the operand is a dense even-ld matrix), B's TPU tiles copied
// as stored ([n][k], LD 36, conflict-free fragment reads) with 16-byte
// cp.async; STAGES-deep ring, one barrier per 32-wide k chunk; the row
// weights scale the accumulator rows at the end.
template <int STAGES>
__host__ __device__ constexpr size_t qform_pipe_smem() {
  return (size_t)STAGES * (64 * kQA + 2 * 32 * kTLD) * sizeof(double);
}

template <class W, int STAGES, bool DENSE16>
__global__ void __launch_bounds__(kGramThreads)
    k_qform_pipe(W win, int64_t rows, int K, const double* __restrict__ B, double* __restrict__ Q,
                 int64_t ldq, const int* skip_flag) {
  if (skip_flag && *skip_flag == 0) return;
  extern __shared__ __align__(16) double qps[];
  __shared__ const double* rp[64];
  __shared__ double rw[64];
  constexpr int SA_N = 64 * kQA, SB_N = 2 * 32 * kTLD;
  const int64_t t0 = (int64_t)blockIdx.x * 64;
  const int L0 = blockIdx.y * 64;
  const int jend = min(K, L0 + 64);
  const int nchunk = (jend + 31) / 32;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp & 1, wn = warp >> 1;
  const int nj = min(4, max(0, (K - (L0 + 32 * wn) + 7) / 8));
  const int JB = L0 >> 5, nbj = (K + 31) / 32;
  if (tid < 64) {
    const int64_t t = t0 + tid;
    rp[tid] = t < rows ? win.row(t) : nullptr;
    rw[tid] = t < rows ? win.weight(t) : 0.0;
  }
  __syncthreads();
  auto issue = [&](int ch) {
    double* sa = qps + (size_t)(ch % STAGES) * (SA_N + SB_N);
    double* sb = sa + SA_N;
    const int k0 = ch * 32;
    if (DENSE16) {
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int e = tid + kGramThreads * u;  // 1024 16-byte chunks
        const int r = e >> 4, c = 2 * (e & 15);
        const double* p = rp[r];
        const bool ok = p && k0 + c < K;
        const unsigned d = (unsigned)__cvta_generic_to_shared(sa + r * kQA + c);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(ok ? p + k0 + c : B),
                     "r"(ok ? 16 : 0)
                     : "memory");
      }
    } else {
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const int e = tid + kGramThreads * u;
        const int r = e >> 5, c = e & 31;
        const double* p = rp[r];
        const bool ok = p && k0 + c < K;
        const unsigned d = (unsigned)__cvta_generic_to_shared(sa + r * kQA + c);
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(d),
                     "l"(ok ? p + W::dir * (k0 + c) : B), "r"(ok ? 8 : 0)
                     : "memory");
      }
    }
    const int I = k0 >> 5;
#pragma unroll
    for (int u = 0; u < 9; ++u) {
      const int e = tid + kGramThreads * u;
      if (e < 2 * 32 * 18) {
        const int sub = e / (32 * 18), rem = e % (32 * 18);
        const int n = rem / 18, kc = rem % 18;
        const int J = JB + sub;
        const bool tok = J < nbj && I <= J;
        const bool ok = tok && n < tpu_w(J, K);
        const double* src = ok ? B + tpu_tile(K, I, J) + (int64_t)n * kTLD + 2 * kc : B;
        const unsigned d = (unsigned)__cvta_generic_to_shared(sb + sub * 32 * kTLD + n * kTLD + 2 * kc);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "r"(ok ? 16 : 0)
                     : "memory");
      }
    }
  };
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
#pragma unroll
  for (int st = 0; st < STAGES - 1; ++st) {
    if (st < nchunk) issue(st);
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  for (int ch = 0; ch < nchunk; ++ch) {
    asm volatile("cp.async.wait_group %0;" ::"n"(STAGES - 2) : "memory");
    __syncthreads();
    if (ch + STAGES - 1 < nchunk) issue(ch + STAGES - 1);
    asm volatile("cp.async.commit_group;" ::: "memory");
    const double* sa = qps + (size_t)(ch % STAGES) * (SA_N + SB_N);
    const double* sb = sa + SA_N + wn * 32 * kTLD;
    auto ksteps = [&](auto full) {
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        double af[4], bf[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) af[i] = sa[(32 * wm + 8 * i + (lane >> 2)) * kQA + 4 * kk + (lane & 3)];
#pragma unroll
        for (int j = 0; j < 4; ++j) bf[j] = sb[(8 * j + (lane >> 2)) * kTLD + 4 * kk + (lane & 3)];
        dmma_4x4<decltype(full)::value>(acc, af, bf, 4, nj);
      }
    };
    if (nj == 4) ksteps(std::true_type{});
    else if (nj > 0) ksteps(std::false_type{});
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int r = 32 * wm + 8 * i + (lane >> 2);
    const int64_t row = t0 + r;
    if (row >= rows) continue;
    const double wr = rw[r];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int col = L0 + 32 * wn + 8 * j + 2 * (lane & 3);
      if (col < K) Q[row * ldq + col] = wr * acc[i][j][0];
      if (col + 1 < K) Q[row * ldq + col + 1] = wr * acc[i][j][1];
    }
  }
}

// dense A rows (weights folded) for the 16-byte pipelined path
template <class W>
__global__ void k_gather_rows(W win, int64_t rows, int K, double* __restrict__ out, int64_t ldo) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.y + threadIdx.y;
  if (t >= rows) return;
  const double* p = win.row(t);
  const double w = win.weight(t);
  double v[8];
  for (int j0 = 0; j0 < K; j0 += 8 * 32) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int j = j0 + threadIdx.x + 32 * u;
      v[u] = j < K ? w * p[W::dir * j] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int j = j0 + threadIdx.x + 32 * u;
      if (j < ldo) out[t * ldo + j] = v[u];
    }
  }
}

}  // namespace tfk
