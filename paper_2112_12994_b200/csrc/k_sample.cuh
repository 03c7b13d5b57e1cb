// k_sample.cuh -- leverage-score sampling without materialising pi or a
// w-length CDF (sketch.cpp:20-59; lsar.cpp:27-36).
//
// After the pass of lag q the scores the next lag samples from are
//   s_{q+1}(i) = s_q(i) + r_q(i)^2 / R_q,
// and the pass has already emitted, per 32-row chunk, A_c = sum s_q and
// B_c = sum r_q^2, plus per-2048-row tile totals.  Sampling lag q+1 is then
//   k_lag_scan : single CTA.  R_q = sum B_t (fixed tree), tile masses
//                S_t = A_t + B_t / R_q, exclusive tile prefix OT, total S.
//   k_draw     : one warp per draw t.  u_t = uniform01 of draw t of
//                Rng(derive_seed(seed, p)) (bit-identical to the reference),
//                v = u_t * S; k-ary search of OT (largest tile with OT <= v),
//                then a sequential scan of the tile's 64 chunk masses and of
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
__global__ void __launch_bounds__(kScanThreads)
    k_lag_scan(const double* __restrict__ tA, const double* __restrict__ tB, int64_t ntile,
               double* __restrict__ OT, double* scal, double* Rhist, double* Shist, int lag,
               int check_r, int* status, int unit_r = 0, const double* r_fixed = nullptr) {
  __shared__ double red[kScanThreads];
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

struct DrawArgs {
  uint64_t seed;        // derive_seed(user_seed, p)
  const uint64_t* seed_ptr;  // nullable: read the seed from device memory (graph replays)
  int64_t c;
  const double* scal;   // R, S
  const double* OT;
  int64_t ntile;
  const double* tA;
  const double* tB;
  const double* chunkA;
  const double* chunkB;
  const double* s;      // s_q
  const double* r;      // r_q (nullable: plain scores, r = 0)
  int64_t w;
  int64_t* idx;
  double* wts;
  // row-sharded mode: this shard holds the global CDF segment
  // [offset, offset + S); draws outside it are skipped (accept[t] = 0)
  int shard;
  double s_total;
  double offset;
  int is_last;
  int* accept;
};

constexpr int kDrawThreads = 256;

__global__ void __launch_bounds__(kDrawThreads) k_draw(DrawArgs a) {
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int64_t t = (int64_t)blockIdx.x * (kDrawThreads / 32) + wib;
  if (t >= a.c) return;
  const double R = a.scal[0], S = a.scal[1];
  const uint64_t seed = a.seed_ptr ? *a.seed_ptr : a.seed;
  double v = rng_uniform01(seed, (uint64_t)t) * (a.shard ? a.s_total : S);
  if (a.shard) {
    v -= a.offset;
    const bool mine = v >= 0.0 && (v < S || a.is_last);
    if (lane == 0) a.accept[t] = mine ? 1 : 0;
    if (!mine) return;
  }
  // ---- tile: largest T with OT[T] <= v ----
  int64_t lo = 0, hi = a.ntile;
  while (hi - lo > 32) {
    const int64_t stride = (hi - lo + 31) / 32;
    const int64_t pos = lo + (int64_t)lane * stride;
    const bool pr = pos < hi && a.OT[pos] <= v;
    int cnt = __popc(__ballot_sync(0xffffffffu, pr));
    if (cnt == 0) cnt = 1;
    lo = lo + (int64_t)(cnt - 1) * stride;
    hi = min(lo + stride, hi);
  }
  {
    const int64_t pos = lo + lane;
    const bool pr = pos < hi && a.OT[pos] <= v;
    int cnt = __popc(__ballot_sync(0xffffffffu, pr));
    if (cnt == 0) cnt = 1;
    lo = lo + cnt - 1;
  }
  int64_t T = lo;
  // a tile with zero mass can only be hit through the end guard: walk back
  // (sketch.cpp:54-55 skips zero-mass rows backwards the same way)
  while (T > 0 && !(a.tA[T] + a.tB[T] / R > 0.0)) --T;
  double v1 = v - a.OT[T];
  // ---- chunk within tile, then row within chunk: warp-parallel CDF search.
  //      Inclusive warp scans of the masses (fixed tree order); the pick is
  //      the first position whose cumulative mass exceeds v with positive
  //      mass (sketch.cpp:45-55 upper_bound + zero-mass skip); past the end,
  //      the last positive entry (end guard).
  const int64_t nchunk = (a.w + kChunk - 1) / kChunk;
  const int64_t cb = T * kChunksPerTile;
  const int nch = (int)min((int64_t)kChunksPerTile, nchunk - cb);
  int chosen = -1;
  double vrow = 0.0;
  {
    double base = 0.0;
    int lastpos = -1;
    for (int h = 0; h < 2 && chosen < 0; ++h) {
      const int k = 32 * h + lane;
      const double m = k < nch ? a.chunkA[cb + k] + a.chunkB[cb + k] / R : 0.0;
      const double inc = base + warp_incl_scan(m);
      const unsigned hit = __ballot_sync(0xffffffffu, inc > v1 && m > 0.0);
      const unsigned pos = __ballot_sync(0xffffffffu, m > 0.0);
      if (pos) lastpos = 32 * h + 31 - __clz(pos);
      if (hit) {
        const int src = __ffs(hit) - 1;
        chosen = 32 * h + src;
        vrow = v1 - __shfl_sync(0xffffffffu, inc - m, src);
      }
      base = __shfl_sync(0xffffffffu, inc, 31);
    }
    if (chosen < 0) {
      chosen = lastpos < 0 ? nch - 1 : lastpos;
      vrow = __longlong_as_double(0x7ff0000000000000ll);  // +inf: take last positive row
    }
  }
  const int64_t r0 = (cb + chosen) * kChunk;
  const int64_t row = r0 + lane;
  double mass = 0.0;
  if (row < a.w) {
    if (a.r) {
      const double rv = a.r[row];
      mass = a.s[row] + (rv * rv) / R;
    } else {
      mass = a.s[row] + 0.0 / R;  // same expression as the partials (r = 0)
    }
  }
  const double incr = warp_incl_scan(mass);
  const unsigned hitr = __ballot_sync(0xffffffffu, incr > vrow && mass > 0.0);
  const unsigned posr = __ballot_sync(0xffffffffu, mass > 0.0);
  const int pick = hitr ? __ffs(hitr) - 1 : (posr ? 31 - __clz(posr) : 0);
  const double mp = __shfl_sync(0xffffffffu, mass, pick);
  if (lane == 0) {
    a.idx[t] = r0 + pick;
    a.wts[t] = 1.0 / sqrt((double)a.c * (mp / (a.shard ? a.s_total : S)));
  }
}

}  // namespace tfk
