// k_rh.cuh -- Repeated Halving upfront phase on the GPU
// (repeated_halving.cpp:126-189; generalized leverage repeated_halving.cpp:49-124).
//
// Halving (integer work, bit-exact with the reference).  Level l keeps the
// first half of a partial Fisher-Yates shuffle of level l-1 (step i swaps
// positions i and j_i = i + below(size - i), rng.hpp:59-66) and sorts it.
// The swap sequence is sequential, but its outcome is not: position i ends
// up holding the value that sat at j_i before step i, and that value is
// found by walking back through the earlier steps that targeted the same
// position:
//     q = j_i, bound = i
//     loop: s = largest step < bound with j_s = q;  none -> answer orig[q]
//           q = s, bound = s
// With the steps bucketed by target (count, scan, scatter, tiny per-bucket
// sort) every i resolves independently.  The current level is sorted, so the
// sorted first half is a stream compaction of the level by a "picked" flag.
// Draw i uses counter i of Rng(seed); the below() rejection (probability
// ~bound / 2^64) is detected and then the whole level is redrawn serially.
//
// Gaussian sketch rows (orc_gaussian_apply / rng.hpp:41-56 polar method):
// attempt a uses uniforms 2a, 2a+1; accepted attempt number r yields normals
// 2r (u f) and 2r + 1 (v f).  Acceptance flags + scan place every normal
// without a sequential stream.  log() may differ from glibc by <= 1 ulp.
//
// Generalized leverage of row x against the approximation B (brows x k):
//   sketched:   || G B (B^T B)^-1 x ||^2 / g  = || W^T x ||^2,  W = ((G B) S S^T)^T / sqrt(g)
//   unsketched: x^T (B^T B)^-1 x = || S^T x ||^2
// with S = R^-1 from the CholeskyQR of B (k_cholinv).  This is the same
// quantity the reference forms from its pivoted QR (mix = G Q / sqrt(g),
// z = R^-T P^T x): Q R^-T P^T = B (B^T B)^-1.
#pragma once

#include "common.cuh"
#include "k_gram.cuh"
#include "k_sample.cuh"
#include "k_tpu.cuh"

namespace tfk {

constexpr int kRhThreads = 256;
constexpr int kScanPer = 16;
constexpr int kScanTileN = kRhThreads * kScanPer;  // 4096 elements per scan tile

__device__ __forceinline__ long long warp_incl_scan_ll(long long v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const long long t = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += t;
  }
  return v;
}

// block-wide exclusive scan (kRhThreads threads); returns the exclusive prefix
// of `v`; the block total goes to *tot (shared), valid after return
__device__ __forceinline__ long long block_excl_scan_ll(long long v, long long* tot) {
  __shared__ long long ws[kRhThreads / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const long long inc = warp_incl_scan_ll(v);
  if (lane == 31) ws[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    const long long x = lane < kRhThreads / 32 ? ws[lane] : 0;
    const long long xi = warp_incl_scan_ll(x);
    if (lane < kRhThreads / 32) ws[lane] = xi - x;
    if (lane == 31) *tot = xi;
  }
  __syncthreads();
  const long long r = ws[warp] + inc - v;
  __syncthreads();
  return r;
}

// ---- scan of int32 values: tile sums -> top scan -> apply ----
__global__ void __launch_bounds__(kRhThreads)
    k_scan_tile_sums(const int* __restrict__ in, int64_t n, long long* __restrict__ tsum) {
  __shared__ long long tot;
  const int64_t base = (int64_t)blockIdx.x * kScanTileN;
  long long acc = 0;
#pragma unroll
  for (int u = 0; u < kScanPer; ++u) {
    const int64_t i = base + (int64_t)u * kRhThreads + threadIdx.x;
    if (i < n) acc += in[i];
  }
  block_excl_scan_ll(acc, &tot);
  if (threadIdx.x == 0) tsum[blockIdx.x] = tot;
}

// single CTA: in-place exclusive scan of the tile sums; total -> *total
__global__ void __launch_bounds__(1024) k_scan_top(long long* __restrict__ tsum, int64_t nt,
                                                   long long* __restrict__ total) {
  __shared__ long long ws[32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t seg = (nt + 1023) / 1024;
  const int64_t b = min(nt, (int64_t)tid * seg), e = min(nt, b + seg);
  long long s = 0;
  for (int64_t t = b; t < e; ++t) s += tsum[t];
  const long long inc = warp_incl_scan_ll(s);
  if (lane == 31) ws[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    const long long x = ws[lane];
    const long long xi = warp_incl_scan_ll(x);
    ws[lane] = xi - x;
    if (lane == 31) *total = xi;
  }
  __syncthreads();
  long long off = ws[warp] + inc - s;
  for (int64_t t = b; t < e; ++t) {
    const long long v = tsum[t];
    tsum[t] = off;
    off += v;
  }
}

// per-tile exclusive scan; f(i, excl, value) for every i < n (thread-contiguous order)
template <class F>
__global__ void __launch_bounds__(kRhThreads)
    k_scan_apply(const int* __restrict__ in, int64_t n, const long long* __restrict__ toff, F f) {
  __shared__ long long tot;
  const int64_t base = (int64_t)blockIdx.x * kScanTileN + (int64_t)threadIdx.x * kScanPer;
  int v[kScanPer];
  long long s = 0;
#pragma unroll
  for (int u = 0; u < kScanPer; ++u) {
    v[u] = base + u < n ? in[base + u] : 0;
    s += v[u];
  }
  long long run = toff[blockIdx.x] + block_excl_scan_ll(s, &tot);
#pragma unroll
  for (int u = 0; u < kScanPer; ++u) {
    if (base + u < n) f(base + u, run, v[u]);
    run += v[u];
  }
}

// ---- halving ----
__device__ __forceinline__ uint64_t below_limit(uint64_t bound) {
  const uint64_t mx = ~0ull;
  return mx - mx % bound;
}

__global__ void k_halve_draw(uint64_t seed, int64_t size, int64_t half, int* __restrict__ J,
                             int* __restrict__ reject) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < half;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t bound = (uint64_t)(size - i);
    const uint64_t x = rng_draw(seed, (uint64_t)i);
    if (x >= below_limit(bound)) *reject = 1;
    J[i] = (int)(i + (int64_t)(x % bound));
  }
}

// rare path: some draw was rejected -> redraw the level with the sequential counter
__global__ void k_halve_draw_serial(uint64_t seed, int64_t size, int64_t half, int* __restrict__ J,
                                    const int* __restrict__ reject) {
  if (*reject == 0 || threadIdx.x != 0 || blockIdx.x != 0) return;
  uint64_t t = 0;
  for (int64_t i = 0; i < half; ++i) {
    const uint64_t bound = (uint64_t)(size - i), lim = below_limit(bound);
    uint64_t x;
    do {
      x = rng_draw(seed, t++);
    } while (x >= lim);
    J[i] = (int)(i + (int64_t)(x % bound));
  }
}

__global__ void k_halve_count(const int* __restrict__ J, int64_t half, int* __restrict__ cnt) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < half;
       i += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(cnt + J[i], 1);
}

struct StartF {
  int* start;
  __device__ void operator()(int64_t i, long long excl, int) const { start[i] = (int)excl; }
};

__global__ void k_halve_scatter(const int* __restrict__ J, int64_t half, const int* __restrict__ start,
                                int* __restrict__ fill, int* __restrict__ bk) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < half;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int j = J[i];
    bk[start[j] + atomicAdd(fill + j, 1)] = (int)i;
  }
}

__global__ void k_halve_bucket_sort(const int* __restrict__ cnt, const int* __restrict__ start,
                                    int64_t size, int* __restrict__ bk) {
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < size;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int c = cnt[q];
    if (c < 2) continue;
    int* b = bk + start[q];
    for (int a = 1; a < c; ++a) {
      const int v = b[a];
      int k = a - 1;
      while (k >= 0 && b[k] > v) {
        b[k + 1] = b[k];
        --k;
      }
      b[k + 1] = v;
    }
  }
}

__global__ void k_halve_resolve(const int* __restrict__ J, int64_t half, const int* __restrict__ cnt,
                                const int* __restrict__ start, const int* __restrict__ bk,
                                int* __restrict__ picked) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < half;
       i += (int64_t)gridDim.x * blockDim.x) {
    int q = J[i], bound = (int)i;
    for (;;) {
      const int c = cnt[q], st = start[q];
      int best = -1;
      for (int k = 0; k < c; ++k) {
        const int s = bk[st + k];
        if (s < bound) best = s;
        else break;
      }
      if (best < 0) break;
      q = best;
      bound = best;
    }
    picked[q] = 1;
  }
}

// next level = cur[q] for picked q, in position order (cur sorted -> next sorted)
struct CompactF {
  const int64_t* cur;  // nullable: identity (level 0)
  int64_t* next;
  __device__ void operator()(int64_t i, long long excl, int v) const {
    if (v) next[excl] = cur ? cur[i] : i;
  }
};

// ---- polar normals ----
__device__ __forceinline__ void polar_attempt(uint64_t seed, int64_t a, double& u, double& v,
                                              double& s) {
  u = __dadd_rn(-1.0, __dmul_rn(2.0, rng_uniform01(seed, 2 * (uint64_t)a)));
  v = __dadd_rn(-1.0, __dmul_rn(2.0, rng_uniform01(seed, 2 * (uint64_t)a + 1)));
  s = __dadd_rn(__dmul_rn(u, u), __dmul_rn(v, v));
}

__global__ void k_polar_flags(uint64_t seed, int64_t attempts, int* __restrict__ ok) {
  for (int64_t a = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; a < attempts;
       a += (int64_t)gridDim.x * blockDim.x) {
    double u, v, s;
    polar_attempt(seed, a, u, v, s);
    ok[a] = (s < 1.0 && s != 0.0) ? 1 : 0;
  }
}

struct PolarF {
  uint64_t seed;
  int64_t count;  // normals wanted
  double* out;
  __device__ void operator()(int64_t a, long long r, int v) const {
    if (!v) return;
    const int64_t q = 2 * (int64_t)r;
    if (q >= count) return;
    double u, vv, s;
    polar_attempt(seed, a, u, vv, s);
    const double f = __dsqrt_rn(__ddiv_rn(-2.0 * log(s), s));
    out[q] = __dmul_rn(u, f);
    if (q + 1 < count) out[q + 1] = __dmul_rn(vv, f);
  }
};

// ---- sketch matrices ----
// rows of the concatenation [N | B] (N: rows x g row-major normals, B: approx rows)
template <class L>
struct ConcatRowsT {
  const double* nm;
  int g;
  L fr;
  __device__ __forceinline__ double operator()(int64_t t, int col) const {
    return col < g ? nm[t * g + col] : fr(t, col - g);
  }
};
using ConcatRows = ConcatRowsT<FwdRows>;

// a dense row-major matrix with one appended zero column (the rank check of a
// reference matrix through the pivoted Cholesky, which carries a target column)
struct DenseRowsZ {
  const double* q;
  int64_t ld;
  int k;
  __device__ __forceinline__ double operator()(int64_t t, int col) const { return col < k ? q[t * ld + col] : 0.0; }
};

// H0[i][l] = sum_{a <= l} GB[i][a] S[a][l]; GB[i][a] = Gp(i, g + a) (TPU, Kp = g + K)
__global__ void k_rh_h0(const double* __restrict__ Gp, int Kp, int g, const double* __restrict__ S,
                        int K, double* __restrict__ H0) {
  const int64_t tot = (int64_t)g * K;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < tot;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(e / K), l = (int)(e % K);
    double acc = 0.0;
    for (int a = 0; a <= l; ++a) acc = fma(Gp[tpu_idx(Kp, i, g + a)], S[tpu_idx(K, a, l)], acc);
    H0[e] = acc;
  }
}

// W[a][i] = (sum_{l >= a} H0[i][l] S[a][l]) / sqrt(g)   (K x g row-major)
__global__ void k_rh_w(const double* __restrict__ H0, const double* __restrict__ S, int K, int g,
                       double* __restrict__ W) {
  const int64_t tot = (int64_t)g * K;
  const double sg = sqrt((double)g);
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < tot;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int a = (int)(e / g), i = (int)(e % g);
    double acc = 0.0;
    for (int l = a; l < K; ++l) acc = fma(H0[(int64_t)i * K + l], S[tpu_idx(K, a, l)], acc);
    W[e] = acc / sg;
  }
}

// ---- row scores: out[t] = || x_t W ||^2 ----
struct WinRows {  // unweighted forward rows y[b_t .. b_t + K); idx nullable -> b_t = t
  const double* y;
  const int64_t* idx;
  __device__ __forceinline__ double operator()(int64_t t, int col) const {
    return y[(idx ? idx[t] : t) + col];
  }
  __device__ __forceinline__ const double* row(int64_t t) const { return y + (idx ? idx[t] : t); }
};
struct DenseW {
  const double* w;
  int ld;
  __device__ __forceinline__ double operator()(int k, int n) const { return w[(int64_t)k * ld + n]; }
};
struct TpuW {
  const double* S;
  int K;
  __device__ __forceinline__ double operator()(int k, int n) const {
    return k <= n ? S[tpu_idx(K, k, n)] : 0.0;
  }
};

constexpr size_t kRowsqSmem = (64 * kQA + 32 * kSJ) * sizeof(double);

// out[t] = || x_t W ||^2 over column tiles of W (K x N); 8-wide fragments
// past column N are skipped (warp-uniform).
template <class L, class WL, bool UPPER>
__global__ void __launch_bounds__(kGramThreads)
    k_rowsq(L ld, int64_t rows, int K, WL wl, int N, double* __restrict__ out) {
  extern __shared__ __align__(16) double rq_smem[];
  double(*SA)[64][kQA] = reinterpret_cast<double(*)[64][kQA]>(rq_smem);
  double(*SW)[32][kSJ] = reinterpret_cast<double(*)[32][kSJ]>(rq_smem + 64 * kQA);
  __shared__ double red[2][64];
  const int64_t t0 = (int64_t)blockIdx.x * 64;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp & 1, wn = warp >> 1;
  const int cc = tid & 31, rr0 = tid >> 5;
  const int ll = tid & 63, c0 = tid >> 6;
  double rs[4] = {0.0, 0.0, 0.0, 0.0};
  for (int N0 = 0; N0 < N; N0 += 64) {
    const int nj = min(4, max(0, (N - (N0 + 32 * wn) + 7) / 8));
    double acc[4][4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    const int kend = UPPER ? min(K, N0 + 64) : K;
    for (int k0 = 0; k0 < kend; k0 += 32) {
#pragma unroll
      for (int s = 0; s < 16; ++s) {
        const int64_t row = t0 + rr0 + 4 * s;
        SA[0][rr0 + 4 * s][cc] = (row < rows && k0 + cc < K) ? ld(row, k0 + cc) : 0.0;
      }
#pragma unroll
      for (int s = 0; s < 16; ++s) {
        const int c = k0 + c0 + 2 * s;
        SW[0][c0 + 2 * s][ll] = (c < K && N0 + ll < N) ? wl(c, N0 + ll) : 0.0;
      }
      __syncthreads();
      auto ksteps = [&](auto full) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          double af[4], bf[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) af[i] = SA[0][32 * wm + 8 * i + (lane >> 2)][4 * kk + (lane & 3)];
#pragma unroll
          for (int j = 0; j < 4; ++j) bf[j] = SW[0][4 * kk + (lane & 3)][32 * wn + 8 * j + (lane >> 2)];
          dmma_4x4<decltype(full)::value>(acc, af, bf, 4, nj);
        }
      };
      if (nj == 4) ksteps(std::true_type{});
      else if (nj > 0) ksteps(std::false_type{});
      __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) rs[i] = fma(acc[i][j][0], acc[i][j][0], fma(acc[i][j][1], acc[i][j][1], rs[i]));
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    rs[i] += __shfl_xor_sync(0xffffffffu, rs[i], 1);
    rs[i] += __shfl_xor_sync(0xffffffffu, rs[i], 2);
    if ((lane & 3) == 0) red[wn][32 * wm + 8 * i + (lane >> 2)] = rs[i];
  }
  __syncthreads();
  if (tid < 64 && t0 + tid < rows) out[t0 + tid] = red[0][tid] + red[1][tid];
}

// Row scores over CONSECUTIVE windows x_t = y[t .. t + K) (level 0 and the
// final unsketched pass, i.e. every row of the window): the 64-row A tile of a
// row block is the Hankel matrix of the 64 + K series values it spans, so a
// block costs one short vector load instead of 64 x K gathered values.
// Persistent CTAs, one per (column tile of W, SM): the CTA keeps its K x 64
// slice of W resident in shared memory and streams row blocks, prefetching the
// next block's series segment with cp.async while DMMA runs.  Per-tile partial
// sums of squares go to part[tile][row]; k_rowsq_combine adds them in order.
constexpr int kHkLd = 68;       // W slice row stride (doubles)
constexpr int kHkRows = 128;    // rows per block (8 warps: 4 row x 2 column warp tiles)
constexpr int kHkThreads = 256;

__host__ __device__ inline int hk_kpad(int K) { return (K + 7) & ~7; }  // k runs in steps of 8
__host__ inline size_t rowsq_hankel_smem(int K) {
  return ((size_t)hk_kpad(K) * kHkLd + 2 * (size_t)(kHkRows + hk_kpad(K) + 48)) * sizeof(double);
}

// CTAs per column tile are proportional to the tile's DMMA work (narrow last
// tiles and the triangular final pass would otherwise leave SMs idle)
struct HkPlan {
  int ntiles;
  int first[9];  // CTA range of tile j: [first[j], first[j + 1])
};

template <class WL, bool UPPER>
__global__ void __launch_bounds__(kHkThreads)
    k_rowsq_hankel(const double* __restrict__ y, int64_t n, int64_t rows, int K, WL wl, int N, HkPlan plan,
                   double* __restrict__ part) {
  extern __shared__ __align__(16) double hk[];
  __shared__ double red[2][kHkRows];
  const int kp = hk_kpad(K);
  const int seg = kHkRows + kp + 48;
  double* Wt = hk;
  double* yb = hk + (size_t)kp * kHkLd;
  int tile = 0;
  while (tile + 1 < plan.ntiles && (int)blockIdx.x >= plan.first[tile + 1]) ++tile;
  const int cta = blockIdx.x - plan.first[tile], nct = plan.first[tile + 1] - plan.first[tile];
  const int N0 = tile * 64;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp & 3, wn = warp >> 2;
  const int nj = min(4, max(0, (N - (N0 + 32 * wn) + 7) / 8));
  const int kend = UPPER ? min(kp, hk_kpad(min(K, N0 + 64))) : kp;
  for (int e = tid; e < kp * 64; e += kHkThreads) {
    const int k = e >> 6, c = e & 63;
    Wt[k * kHkLd + c] = (k < K && N0 + c < N) ? wl(k, N0 + c) : 0.0;
  }
  const int64_t nblk = (rows + kHkRows - 1) / kHkRows;
  auto fetch = [&](int64_t b, double* dst) {
    const int64_t t0 = b * kHkRows;
    for (int x = tid; x < seg; x += kHkThreads) {
      const int64_t gi = t0 + x;
      const bool ok = gi < n;
      const unsigned d = (unsigned)__cvta_generic_to_shared(dst + x);
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(d), "l"(y + (ok ? gi : 0)),
                   "r"(ok ? 8 : 0)
                   : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  int buf = 0;
  if (cta < nblk) fetch(cta, yb);
  for (int64_t b = cta; b < nblk; b += nct) {
    const int64_t bn = b + nct;
    if (bn < nblk) fetch(bn, yb + (buf ^ 1) * seg);
    if (bn < nblk) asm volatile("cp.async.wait_group 1;" ::: "memory");
    else asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncthreads();
    const double* ys = yb + buf * seg;
    double acc[4][4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    // Hankel A fragments: row 8 i + r at column k equals row 8 (i + 1) + r at
    // column k - 8, so two register windows (k = 0 and k = 4 mod 8) advance
    // with one new shared-memory load each per 8 columns
    auto ksteps = [&](auto full) {
      constexpr bool F = decltype(full)::value;
      const int rbase = 32 * wm + (lane >> 2) + (lane & 3);
      double ae[4], ao[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        ae[i] = ys[rbase + 8 * i];
        ao[i] = ys[rbase + 8 * i + 4];
      }
#pragma unroll 2
      for (int k = 0; k < kend; k += 8) {
        double bf[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) bf[j] = Wt[(k + (lane & 3)) * kHkLd + 32 * wn + 8 * j + (lane >> 2)];
        const double ae_n = ys[rbase + k + 32];
        const double ao_n = ys[rbase + k + 36];
        dmma_4x4<F>(acc, ae, bf, 4, nj);
#pragma unroll
        for (int j = 0; j < 4; ++j) bf[j] = Wt[(k + 4 + (lane & 3)) * kHkLd + 32 * wn + 8 * j + (lane >> 2)];
        dmma_4x4<F>(acc, ao, bf, 4, nj);
#pragma unroll
        for (int i = 0; i < 3; ++i) {
          ae[i] = ae[i + 1];
          ao[i] = ao[i + 1];
        }
        ae[3] = ae_n;
        ao[3] = ao_n;
      }
    };
    if (nj == 4) ksteps(std::true_type{});
    else if (nj > 0) ksteps(std::false_type{});
    if ((lane & 3) == 0 || true) {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        double v = 0.0;
#pragma unroll
        for (int j = 0; j < 4; ++j) v = fma(acc[i][j][0], acc[i][j][0], fma(acc[i][j][1], acc[i][j][1], v));
        v += __shfl_xor_sync(0xffffffffu, v, 1);
        v += __shfl_xor_sync(0xffffffffu, v, 2);
        if ((lane & 3) == 0) red[wn][32 * wm + 8 * i + (lane >> 2)] = v;
      }
    }
    __syncthreads();
    const int64_t t0 = b * kHkRows;
    if (tid < kHkRows && t0 + tid < rows) part[(size_t)tile * rows + t0 + tid] = red[0][tid] + red[1][tid];
    buf ^= 1;
  }
}

// Narrow last column tile of W (N - N0 <= kTailMax columns, e.g. the 129th
// sketch row g = ceil(8 ln m)): out[t] (+)= sum_j (x_t . W[:, j])^2 on the
// CUDA cores, one row per thread (K fmas per column), W's tail columns in
// shared memory.  A DMMA tile pass for one or a few columns would pay a whole
// tile's loads and barriers for 1/8 of a fragment of work.
constexpr int kTailMax = 16;
// MT: max tail columns, RW: rows per thread (32 apart: coalesced loads; one
// W read serves RW rows); instantiated as <2, 8>, <12, 4>, <16, 2>
template <class L, class WL, int MT, int RW>
__global__ void __launch_bounds__(256) k_rowsq_tail(L ld, int64_t rows, int K, WL wl, int N0, int N,
                                                    double* __restrict__ out, int add) {
  extern __shared__ double wtail[];  // [K][T]
  const int T = N - N0;
  for (int e = threadIdx.x; e < K * T; e += blockDim.x) wtail[e] = wl(e / T, N0 + e % T);
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t nblk = (rows + 32 * RW - 1) / (32 * RW);  // 256-row warp blocks
  for (int64_t wb = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp; wb < nblk;
       wb += (int64_t)gridDim.x * (blockDim.x >> 5)) {
    const int64_t t0 = wb * 32 * RW + lane;
    const double* row[RW];
#pragma unroll
    for (int r = 0; r < RW; ++r) row[r] = ld.row(min(t0 + 32 * r, rows - 1));
    double acc[RW][MT];
#pragma unroll
    for (int r = 0; r < RW; ++r)
#pragma unroll
      for (int j = 0; j < MT; ++j) acc[r][j] = 0.0;
    for (int k = 0; k < K; ++k) {
      double x[RW];
#pragma unroll
      for (int r = 0; r < RW; ++r) x[r] = __ldg(row[r] + k);
#pragma unroll
      for (int j = 0; j < MT; ++j) {
        if (j < T) {
          const double wv = wtail[k * T + j];
#pragma unroll
          for (int r = 0; r < RW; ++r) acc[r][j] = fma(x[r], wv, acc[r][j]);
        }
      }
    }
#pragma unroll
    for (int r = 0; r < RW; ++r) {
      const int64_t t = t0 + 32 * r;
      if (t < rows) {
        double v = 0.0;
#pragma unroll
        for (int j = 0; j < MT; ++j)
          if (j < T) v = fma(acc[r][j], acc[r][j], v);
        out[t] = add ? out[t] + v : v;
      }
    }
  }
}

__global__ void k_rowsq_combine(const double* __restrict__ part, int64_t rows, int ntiles,
                                double* __restrict__ out) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < rows;
       t += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int j = 0; j < ntiles; ++j) s += part[(size_t)j * rows + t];
    out[t] = s;
  }
}

// next approximation rows: idx = cur[sidx] (cur nullable -> identity), weights = sw
__global__ void k_rh_compose(const int64_t* __restrict__ sidx, const double* __restrict__ sw,
                             const int64_t* __restrict__ cur, int64_t sc, int64_t* __restrict__ aidx,
                             double* __restrict__ aw) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < sc;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t q = sidx[t];
    aidx[t] = cur ? cur[q] : q;
    aw[t] = sw[t];
  }
}

__global__ void k_iota(int64_t* __restrict__ p, int64_t n) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x)
    p[t] = t;
}

// the accepted-attempt total must cover the normals wanted
__global__ void k_check_normals(const long long* total, int64_t pairs, int* status) {
  if (*total < pairs) raise_status(status, kErrNumerical, 0, kReasonSketchStream);
}

__global__ void k_fill(double* __restrict__ p, int64_t n, double v) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x)
    p[t] = v;
}

}  // namespace tfk
