// k_sample.cuh -- leverage-score sampling without materialising pi or a
// w-length CDF (sketch.cpp:20-59; lsar.cpp:27-36).
//
// After the pass of lag q the scores the next lag samples from are
//   s_{q+1}(i) = s_q(i) + r_q(i)^2 / R_q,
// and the pass has already emitted, per 32-row chunk, A_c = sum s_q and
// B_c = sum r_q^2, plus per-2048-row tile totals.  Sampling lag q+1 is then
//   k_lag_scan : single CTA.  R_q = sum B_t (fixed tree), tile masses
//                S_t = A_t + B_t / R_q, exclusive tile prefix OT, total S.
//                It also fills a guide table: the first tile of each of G
//                equal buckets of [0, S).
//   k_draw     : one group of 8 lanes per draw t (4 draws per warp).  u_t = uniform01 of draw t of
//                Rng(derive_seed(seed, p)) (bit-identical to the reference),
//                v = u_t * S; the guide table brackets the tile (largest
//                tile with OT <= v; usually one 32-wide probe), then
//                warp scans of the tile's 64 chunk masses and of
//                the chunk's 32 row masses -- "first cumulative mass > v",
//                i.e. std::upper_bound on the CDF.  Row masses are computed
//                with the exact expression the next pass stores, so the
//                weight 1/sqrt(c * s(i)/S) matches the stored scores.
// Rounding differs from the reference's sequential CDF only at the ~1e-16
// level; draws are distributionally identical (and identical in practice).
#pragma once

#include "common.cuh"
#include "k_pass.cuh"

namespace tfk {

enum : int { kErrNone = 0, kErrUsage = 1, kErrData = 2, kErrNumerical = 3 };

// status[0] = first error code, status[1] = lag of that error, status[2] = reason id
__device__ __forceinline__ void raise_status(int* status, int code, int lag, int reason) {
  if (atomicCAS(status, 0, code) == 0) {
    status[1] = lag;
    status[2] = reason;
  }
}

// reason ids (host maps them to the reference's messages)
enum : int {
  kReasonZeroResidual = 1,  // lsar.cpp:21-23
  kReasonNegativeScore = 2, // lsar.cpp:29-31
  kReasonZeroScoreSum = 3,  // lsar.cpp:33
  kReasonCholFail = 4,      // compressed solve failed
  kReasonRankDeficient = 5, // RH reference matrix rank deficient (repeated_halving.cpp:57-64)
  kReasonZeroWindow = 6,    // lsar.cpp:13 all-zero window
  kReasonSketchStream = 7,  // polar normal stream shorter than the sketch (never in practice)
};

constexpr int kScanThreads = 1024;

// scal[0] = R_q, scal[1] = S (total mass for lag q+1)
// Guide table for the draws' tile search (inverse transform with a guide
// table): G equal buckets of [0, S), bucket(x) = min(G - 1, (int)(x * (G / S))),
// first[b] = smallest tile T with bucket(OT[T]) >= b (first[G] = ntile).
// bucket() is monotone, so a draw v in bucket b has its tile in
// [max(0, first[b] - 1), first[b + 1]) -- exact, no tolerance.
constexpr int kGuideMax = 8192;
__host__ __device__ inline int guide_buckets(int64_t ntile) { return (int)min(ntile, (int64_t)kGuideMax); }
__device__ __forceinline__ int guide_bucket(double x, double gscale, int G) {
  const double f = x * gscale;
  return f >= (double)(G - 1) ? G - 1 : (f > 0.0 ? (int)f : 0);
}

__global__ void __launch_bounds__(kScanThreads)
    k_lag_scan(const double* __restrict__ tA, const double* __restrict__ tB, int64_t ntile,
               double* __restrict__ OT, double* scal, double* Rhist, double* Shist, int lag,
               int check_r, int* status, int unit_r = 0, const double* r_fixed = nullptr,
               int* __restrict__ guide = nullptr, int64_t bs_tile = 0, int bs_hist = 0) {
  __shared__ double red[kScanThreads];
  if (blockIdx.x) {  // batched sweeps: series b = blockIdx.x (4 scalars, 4 status words each)
    const int64_t b = blockIdx.x;
    tA += b * bs_tile;
    tB += b * bs_tile;
    OT += b * bs_tile;
    scal += 4 * b;
    status += 4 * b;
    if (Rhist) Rhist += b * bs_hist;
    if (Shist) Shist += b * bs_hist;
    if (guide) guide += b * (guide_buckets(ntile) + 1);
  }
  __shared__ double wsum[32];
  const int tid = threadIdx.x;
  const int64_t seg = (ntile + kScanThreads - 1) / kScanThreads;
  const int64_t b = min(ntile, (int64_t)tid * seg), e = min(ntile, b + seg);
  double sb = 0.0;
  for (int64_t t = b; t < e; ++t) sb += tB[t];
  red[tid] = sb;
  __syncthreads();
  for (int o = kScanThreads / 2; o > 0; o >>= 1) {
    if (tid < o) red[tid] = red[tid] + red[tid + o];
    __syncthreads();
  }
  const double R = r_fixed ? *r_fixed : (unit_r ? 1.0 : red[0]);
  __syncthreads();
  double ss = 0.0;
  for (int64_t t = b; t < e; ++t) ss += tA[t] + tB[t] / R;
  // block exclusive scan of the segment sums (fixed order)
  const int lane = tid & 31, warp = tid >> 5;
  const double inc = warp_incl_scan(ss);
  double ex = __shfl_up_sync(0xffffffffu, inc, 1);
  if (lane == 0) ex = 0.0;
  if (lane == 31) wsum[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    const double wi = warp_incl_scan(wsum[lane]);
    double we = __shfl_up_sync(0xffffffffu, wi, 1);
    if (lane == 0) we = 0.0;
    __syncwarp();
    wsum[lane] = we;
    if (lane == 31) red[0] = wi;
  }
  __syncthreads();
  double off = wsum[warp] + ex;
  const double S = red[0];
  for (int64_t t = b; t < e; ++t) {
    OT[t] = off;
    off += tA[t] + tB[t] / R;
  }
  if (guide) {
    // each thread scatters the bucket starts of its own tiles: tile t is the
    // first tile of buckets (bucket(OT[t-1]), bucket(OT[t])]
    __shared__ int last_b[kScanThreads];
    const int G = guide_buckets(ntile);
    const double gscale = S > 0.0 ? (double)G / S : 0.0;
    last_b[tid] = e > b ? guide_bucket(OT[e - 1], gscale, G) : -2;
    __syncthreads();
    if (e > b) {
      int bprev = tid > 0 ? last_b[tid - 1] : -1;
      for (int64_t t = b; t < e; ++t) {
        const int bt = guide_bucket(OT[t], gscale, G);
        for (int k = bprev + 1; k <= bt; ++k) guide[k] = (int)t;
        bprev = bt;
      }
      if (e == ntile)
        for (int k = bprev + 1; k <= G; ++k) guide[k] = (int)ntile;
    }
  }
  if (tid == 0) {
    scal[0] = R;
    scal[1] = S;
    if (Rhist) Rhist[lag] = R;
    if (Shist) Shist[lag + 1] = S;
    if (check_r && R == 0.0)
      raise_status(status, kErrNumerical, lag + 1, lag == 0 ? kReasonZeroWindow : kReasonZeroResidual);
    if (!(S >= 0.0) || !(R >= 0.0)) raise_status(status, kErrUsage, lag + 1, kReasonNegativeScore);
    else if (S == 0.0) raise_status(status, kErrNumerical, lag + 1, kReasonZeroScoreSum);
  }
}

// Row masses under the FFT pass's deferred folding (k_fft.cuh, kFftSlots):
// s_{q+1}(row) = s(row) + the row group's pending r_j^2 / R_j in lag order --
// the fma sequence the classic fold applies once per lag (bit-identical).
// K <= 1: classic state (s_q, r_q in place; DrawArgs::s / r).
struct PendState {
  int K;            // superblock groups
  int navail;       // residual arrays in pend (oldest first)
  int64_t sbrows;   // rows per superblock
  int64_t sbgrid;   // the FFT pass's grid: superblock sb is in group (sb + sb / sbgrid) mod K
  const double* pend[4];
  const double* Rp;  // R of the pend lags
  int npg[4];        // per group: the newest npg[g] arrays are not yet folded into s
};
__device__ __forceinline__ double pend_mass(const PendState& ps, const double* __restrict__ s, int64_t row) {
  double m = s[row];
  const int64_t sb = row / ps.sbrows;
  const int g = (int)((sb + sb / ps.sbgrid) % ps.K);
  const int np = g == 0 ? ps.npg[0] : g == 1 ? ps.npg[1] : g == 2 ? ps.npg[2] : ps.npg[3];
  const int k0 = ps.navail - np;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    if (k >= k0 && k < ps.navail) {
      const double rv = ps.pend[k][row];
      m = fma(rv * rv, 1.0 / ps.Rp[k], m);
    }
  }
  return m;
}

struct DrawArgs {
  uint64_t seed;        // derive_seed(user_seed, p)
  const uint64_t* seed_ptr;  // nullable: read the seed from device memory (graph replays)
  int64_t c;
  const double* scal;   // R, S
  const double* OT;
  const int* guide;     // k_lag_scan's guide table (nullable: full k-ary search)
  int64_t ntile;
  const double* tA;
  const double* tB;
  const double* chunkA;
  const double* chunkB;
  const double* s;      // s_q
  const double* r;      // r_q (nullable: plain scores, r = 0)
  PendState ps;         // ps.K > 1: deferred folding (s, r above unused for the row masses)
  int64_t w;
  int64_t* idx;
  double* wts;
  // row-sharded mode: par = (R, S_total, lo, hi) on the device
  // (k_shard_scal); draw t belongs to this shard iff lo <= u_t S_total < hi
  // (the shards' prefix masses in rank order, identical on every rank: each
  // draw lands in exactly one shard) and is resolved at v = u_t S_total - lo
  // in the local CDF; accept[t] records it
  int shard;
  const double* par;
  int* accept;
  // batched sweeps: series b = blockIdx.y at base + b * stride
  int64_t bs_w, bs_chunk, bs_tile, bs_seed;
};

constexpr int kDrawThreads = 256;
constexpr int kDrawL = 8;                    // lanes per draw
constexpr int kDrawPerWarp = 32 / kDrawL;    // draws in flight per warp
constexpr int kDrawPerCta = kDrawThreads / kDrawL;

// lane-group primitives (groups of kDrawL lanes; every lane of a group takes
// the same path, so the group mask is exact)
struct DrawGroup {
  unsigned mask;
  int sl;  // lane within the group
  __device__ __forceinline__ DrawGroup() {
    const int lane = threadIdx.x & 31;
    sl = lane % kDrawL;
    mask = ((1u << kDrawL) - 1u) << (lane - sl);
  }
  __device__ __forceinline__ unsigned ballot(bool p) const {
    return (__ballot_sync(mask, p) & mask) >> ((threadIdx.x & 31) - sl);
  }
  __device__ __forceinline__ double bcast(double x, int src) const { return __shfl_sync(mask, x, src, kDrawL); }
  __device__ __forceinline__ int bcast(int x, int src) const { return __shfl_sync(mask, x, src, kDrawL); }
  __device__ __forceinline__ double incl_scan(double x) const {  // fixed order
#pragma unroll
    for (int o = 1; o < kDrawL; o <<= 1) {
      const double y = __shfl_up_sync(mask, x, o, kDrawL);
      if (sl >= o) x += y;
    }
    return x;
  }
};

// First entry (in order) whose cumulative mass exceeds v with positive mass,
// over NPL consecutive entries per lane (lane sl holds entries NPL sl ..):
// returns the entry index or -1, the mass before it in *before, and the last
// positive entry in *lastpos (-1 if none).  Cumulative sums: per-lane
// sequential prefix + group scan of the lane totals (fixed order).
template <int NPL>
__device__ __forceinline__ int group_pick(const DrawGroup& g, const double (&m)[NPL], double v, double* before,
                                          int* lastpos) {
  double loc[NPL];
  double acc = 0.0;
#pragma unroll
  for (int j = 0; j < NPL; ++j) {
    acc += m[j];
    loc[j] = acc;
  }
  const double excl = g.incl_scan(acc) - acc;
  int jh = -1, jp = -1;
#pragma unroll
  for (int j = NPL - 1; j >= 0; --j) {
    if (m[j] > 0.0) {
      if (excl + loc[j] > v) jh = j;
      if (jp < 0) jp = j;
    }
  }
  const unsigned hit = g.ballot(jh >= 0), pos = g.ballot(jp >= 0);
  *lastpos = pos ? NPL * (31 - __clz(pos)) + g.bcast(jp, 31 - __clz(pos)) : -1;
  if (!hit) return -1;
  const int src = __ffs(hit) - 1;
  const int j = g.bcast(jh, src);
  double b = 0.0;
#pragma unroll
  for (int k = 0; k < NPL; ++k)
    if (k == jh) b = excl + loc[k] - m[k];
  *before = g.bcast(b, src);
  return NPL * src + j;
}

__global__ void __launch_bounds__(kDrawThreads) k_draw(DrawArgs a) {
  const DrawGroup g;
  if (blockIdx.y) {
    const int64_t b = blockIdx.y;
    a.scal += 4 * b;
    a.OT += b * a.bs_tile;
    if (a.guide) a.guide += b * (guide_buckets(a.ntile) + 1);
    a.tA += b * a.bs_tile;
    a.tB += b * a.bs_tile;
    a.chunkA += b * a.bs_chunk;
    a.chunkB += b * a.bs_chunk;
    a.s += b * a.bs_w;
    if (a.r) a.r += b * a.bs_w;
    a.idx += b * a.c;
    a.wts += b * a.c;
    if (a.seed_ptr) a.seed_ptr += b * a.bs_seed;
  }
  const int64_t t = (int64_t)blockIdx.x * kDrawPerCta + (threadIdx.x / kDrawL);
  if (t >= a.c) return;  // group-uniform
  const double R = a.scal[0], S = a.scal[1];
  const double invR = 1.0 / R;
  const uint64_t seed = a.seed_ptr ? *a.seed_ptr : a.seed;
  const double Sw = a.shard ? a.par[1] : S;  // the weights' normaliser: the global score sum
  double v = rng_uniform01(seed, (uint64_t)t) * Sw;
  if (a.shard) {
    const bool mine = v >= a.par[2] && v < a.par[3];
    if (g.sl == 0) a.accept[t] = mine ? 1 : 0;
    if (!mine) return;
    v -= a.par[2];
  }
  // ---- tile: largest T with OT[T] <= v (the guide table brackets it) ----
  int64_t lo = 0, hi = a.ntile;
  if (a.guide) {
    const int G = guide_buckets(a.ntile);
    const int gb = guide_bucket(v, S > 0.0 ? (double)G / S : 0.0, G);
    lo = max(0, a.guide[gb] - 1);
    hi = max(lo + 1, (int64_t)a.guide[gb + 1]);
  }
  while (hi - lo > kDrawL) {  // k-ary narrowing (OT nondecreasing: the predicate is a prefix)
    const int64_t stride = (hi - lo + kDrawL - 1) / kDrawL;
    const int64_t pos = lo + (int64_t)g.sl * stride;
    int cnt = __popc(g.ballot(pos < hi && a.OT[pos] <= v));
    if (cnt == 0) cnt = 1;
    lo = lo + (int64_t)(cnt - 1) * stride;
    hi = min(lo + stride, hi);
  }
  double ot_lo;
  {
    const int64_t pos = lo + g.sl;
    const double ot = pos < hi ? a.OT[pos] : 0.0;
    int cnt = __popc(g.ballot(pos < hi && ot <= v));
    if (cnt == 0) cnt = 1;
    ot_lo = g.bcast(ot, cnt - 1);
    lo = lo + cnt - 1;
  }
  int64_t T = lo;
  double v1 = v - ot_lo;
  // ---- chunk within the tile, then row within the chunk: upper_bound with
  //      the zero-mass skip (sketch.cpp:45-55); past the end, the last
  //      positive entry (end guard).  A tile with zero mass can only be
  //      reached through the end guard (the last tiles): walk back to the
  //      last tile with positive mass and take its last positive entry.
  constexpr int CPL = kChunksPerTile / kDrawL;  // chunks per lane
  const int64_t nchunk = (a.w + kChunk - 1) / kChunk;
  int64_t cb;
  int chosen;
  double vrow;
  for (;;) {
    cb = T * kChunksPerTile;
    const int nch = (int)min((int64_t)kChunksPerTile, nchunk - cb);
    double m[CPL];
#pragma unroll
    for (int j = 0; j < CPL; ++j) {
      const int k = CPL * g.sl + j;
      m[j] = k < nch ? fma(a.chunkB[cb + k], invR, a.chunkA[cb + k]) : 0.0;
    }
    double before = 0.0;
    int lastpos;
    chosen = group_pick<CPL>(g, m, v1, &before, &lastpos);
    if (chosen >= 0) {
      vrow = v1 - before;
      break;
    }
    if (lastpos >= 0 || T == 0) {
      chosen = lastpos < 0 ? nch - 1 : lastpos;
      vrow = __longlong_as_double(0x7ff0000000000000ll);  // +inf: take the last positive row
      break;
    }
    --T;  // zero-mass tile (end guard): walk back
    v1 = __longlong_as_double(0x7ff0000000000000ll);
  }
  constexpr int RPL = kChunk / kDrawL;  // rows per lane
  const int64_t r0 = (cb + chosen) * kChunk;
  double mass[RPL];
#pragma unroll
  for (int j = 0; j < RPL; ++j) {
    const int64_t row = r0 + RPL * g.sl + j;
    mass[j] = 0.0;
    if (row < a.w) {
      if (a.ps.K > 1) {
        mass[j] = pend_mass(a.ps, a.s, row);
      } else if (a.r) {
        const double rv = a.r[row];
        mass[j] = fma(rv * rv, invR, a.s[row]);  // exactly the s_{q+1} the next pass stores
      } else {
        mass[j] = a.s[row];
      }
    }
  }
  double before = 0.0;
  int lastr;
  int pick = group_pick<RPL>(g, mass, vrow, &before, &lastr);
  if (pick < 0) pick = lastr >= 0 ? lastr : 0;
  double mp = 0.0;
#pragma unroll
  for (int j = 0; j < RPL; ++j)
    if (RPL * g.sl + j == pick) mp = mass[j];
  mp = g.bcast(mp, pick / RPL);
  if (g.sl == 0) {
    a.idx[t] = r0 + pick;
    a.wts[t] = 1.0 / sqrt((double)a.c * (mp / Sw));
  }
}

// ---- multi-CTA version of k_lag_scan for long windows (ntile > kScanSingleMax:
//      C4's 488k tiles took 1.3 ms in the single CTA).  Same quantities in a fixed
//      order: R = sum tB (block sums, then the blocks in order), tile masses
//      m_t = tA_t + tB_t / R, OT = exclusive prefix (block-local scans offset by the
//      exclusive prefix of the block totals, each block's total being exactly the
//      last tile's inclusive value, so OT stays nondecreasing across blocks), and
//      the guide table from OT.
constexpr int64_t kScanSingleMax = 16384;
constexpr int kScanBlk = 2 * kScanThreads;  // tiles per block (2 per thread)

// block-wide inclusive scan of one value per thread (fixed order); returns the
// exclusive prefix, *tot = the block total
__device__ __forceinline__ double block_excl_scan(double v, double* wsum, double* tot) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const double inc = warp_incl_scan(v);
  if (lane == 31) wsum[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    const double wi = warp_incl_scan(wsum[lane]);
    __syncwarp();
    wsum[lane] = wi;
  }
  __syncthreads();
  const double before = warp ? wsum[warp - 1] : 0.0;
  *tot = wsum[31];
  return before + (inc - v);
}

__device__ __forceinline__ double tile_mass(const double* tA, const double* tB, int64_t t, int64_t ntile, double R,
                                            int massmode) {
  if (t >= ntile) return 0.0;
  return massmode ? tA[t] + tB[t] / R : tB[t];
}

// per-block totals: massmode 0: sum tB; 1: the scan total of the masses
__global__ void __launch_bounds__(kScanThreads) k_scan_blocks(const double* __restrict__ tA, const double* __restrict__ tB,
                                                              int64_t ntile, const double* __restrict__ scal,
                                                              int massmode, double* __restrict__ part) {
  __shared__ double wsum[32];
  const int64_t t0 = (int64_t)blockIdx.x * kScanBlk + 2 * threadIdx.x;
  const double R = massmode ? scal[0] : 1.0;
  const double v0 = tile_mass(tA, tB, t0, ntile, R, massmode), v1 = tile_mass(tA, tB, t0 + 1, ntile, R, massmode);
  double tot;
  block_excl_scan(v0 + v1, wsum, &tot);
  if (threadIdx.x == 0) part[blockIdx.x] = tot;
}

// one CTA over the block totals.  mode 0: R (or the fixed / unit R) -> scal[0],
// Rhist, the zero-residual check.  mode 1: exclusive prefix of the block totals
// -> boff, S -> scal[1], Shist, the score checks.
__global__ void __launch_bounds__(kScanThreads) k_scan_mid(const double* __restrict__ part, int64_t nb, int mode,
                                                           double* scal, double* Rhist, double* Shist, int lag,
                                                           int check_r, int* status, int unit_r,
                                                           const double* r_fixed, double* __restrict__ boff) {
  __shared__ double wsum[32];
  const int tid = threadIdx.x;
  const int64_t seg = (nb + kScanThreads - 1) / kScanThreads;
  const int64_t b = min(nb, (int64_t)tid * seg), e = min(nb, b + seg);
  double ss = 0.0;
  for (int64_t i = b; i < e; ++i) ss += part[i];
  double tot;
  double off = block_excl_scan(ss, wsum, &tot);
  if (mode == 0) {
    if (tid == 0) {
      const double R = r_fixed ? *r_fixed : (unit_r ? 1.0 : tot);
      scal[0] = R;
      if (Rhist) Rhist[lag] = R;
      if (check_r && R == 0.0)
        raise_status(status, kErrNumerical, lag + 1, lag == 0 ? kReasonZeroWindow : kReasonZeroResidual);
      if (!(R >= 0.0)) raise_status(status, kErrUsage, lag + 1, kReasonNegativeScore);
    }
    return;
  }
  for (int64_t i = b; i < e; ++i) {
    boff[i] = off;
    off += part[i];
  }
  if (tid == 0) {
    const double S = tot;
    scal[1] = S;
    if (Shist) Shist[lag + 1] = S;
    if (!(S >= 0.0)) raise_status(status, kErrUsage, lag + 1, kReasonNegativeScore);
    else if (S == 0.0) raise_status(status, kErrNumerical, lag + 1, kReasonZeroScoreSum);
  }
}

// OT of every tile: the block-local exclusive scan (the same arithmetic as
// k_scan_blocks' total) offset by the block's prefix
__global__ void __launch_bounds__(kScanThreads) k_scan_ot(const double* __restrict__ tA, const double* __restrict__ tB,
                                                          int64_t ntile, const double* __restrict__ scal,
                                                          const double* __restrict__ boff, double* __restrict__ OT) {
  __shared__ double wsum[32];
  const int64_t t0 = (int64_t)blockIdx.x * kScanBlk + 2 * threadIdx.x;
  const double R = scal[0];
  const double v0 = tile_mass(tA, tB, t0, ntile, R, 1), v1 = tile_mass(tA, tB, t0 + 1, ntile, R, 1);
  double tot;
  const double ex = block_excl_scan(v0 + v1, wsum, &tot);
  const double base = boff[blockIdx.x];
  if (t0 < ntile) OT[t0] = base + ex;
  if (t0 + 1 < ntile) OT[t0 + 1] = base + (ex + v0);
}

// guide table from OT: tile t is the first tile of buckets (bucket(OT[t-1]), bucket(OT[t])]
__global__ void k_scan_guide(const double* __restrict__ OT, int64_t ntile, const double* __restrict__ scal,
                             int* __restrict__ guide) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= ntile) return;
  const int G = guide_buckets(ntile);
  const double S = scal[1];
  const double gscale = S > 0.0 ? (double)G / S : 0.0;
  const int bt = guide_bucket(OT[t], gscale, G);
  const int bp = t > 0 ? guide_bucket(OT[t - 1], gscale, G) : -1;
  for (int k = bp + 1; k <= bt; ++k) guide[k] = (int)t;
  if (t == ntile - 1)
    for (int k = bt + 1; k <= G; ++k) guide[k] = (int)ntile;
}

// Row-sharded lag step, part 1: the allgathered (sum s, sum r^2) of every
// shard -> the global R = ||r||^2 (lsar.cpp:17-25), summed in rank order (the
// same arithmetic on every rank).
__global__ void k_shard_R(const double* __restrict__ gath, int world, double* __restrict__ par, double* Rhist,
                          int lag, int* status) {
  double R = 0.0;
  for (int r = 0; r < world; ++r) R += gath[2 * r + 1];
  par[0] = R;
  if (Rhist) Rhist[lag] = R;
  if (R == 0.0) raise_status(status, kErrNumerical, lag + 1, lag == 0 ? kReasonZeroWindow : kReasonZeroResidual);
}

// part 2: the allgathered local CDF totals (each shard's k_lag_scan total with
// the global R) -> the global total S and this shard's segment [lo, hi) of
// the global CDF (prefix in rank order, the last shard's segment open).  Each
// shard resolves its draws against exactly the CDF it built, and one shard
// reproduces the single-GPU sweep bit for bit.
__global__ void k_shard_seg(const double* __restrict__ gS, int world, int rank, double* __restrict__ par,
                            double* Shist, int lag, int* status) {
  double S = 0.0, lo = 0.0, hi = 0.0;
  for (int r = 0; r < world; ++r) {
    if (r == rank) lo = S;
    S += gS[r];
    if (r == rank) hi = S;
  }
  if (rank == world - 1) hi = __longlong_as_double(0x7ff0000000000000ll);
  par[1] = S;
  par[2] = lo;
  par[3] = hi;
  if (Shist) Shist[lag + 1] = S;
  if (!(S > 0.0)) raise_status(status, kErrNumerical, lag + 1, kReasonZeroScoreSum);
}

// Deterministic-index mode with reference indices only: the weight of every
// given row from this lag's own distribution, the exact expression k_draw
// uses (weight 1/sqrt(c * pi_i), sketch.cpp:56-57; mass = s + r^2/R as the
// next pass stores it, or the plain score when r is null).
__global__ void k_fixed_weights(const int64_t* __restrict__ idx, int64_t c, const double* __restrict__ scal,
                                const double* __restrict__ s, const double* __restrict__ r, double* __restrict__ wts,
                                PendState ps) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= c) return;
  const double R = scal[0], S = scal[1];
  const int64_t row = idx[t];
  double mp = s[row];
  if (ps.K > 1) {
    mp = pend_mass(ps, s, row);
  } else if (r) {
    const double rv = r[row];
    mp = fma(rv * rv, 1.0 / R, mp);
  }
  wts[t] = 1.0 / sqrt((double)c * (mp / S));
}

}  // namespace tfk
