// engine.cu -- host orchestration of the B200 LSAR / RH order sweep and the
// C ABI (include/toepfit_b200.h).  One CUDA stream per context; every lag is
// a fixed sequence of kernel launches with no host synchronisation inside the
// sweep (device-side status flags are read once at the end).
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <vector>
#include <type_traits>
#include <mutex>
#include <numeric>
#include <map>

#include "engine.h"
#include "k_bsolve.cuh"
#include "k_cholinv.cuh"
#include "k_exact.cuh"
#include "k_fft.cuh"
#include "k_gen.cuh"
#include "k_gram.cuh"
#include "k_i8gram.cuh"
#include "k_pass.cuh"
#include "k_rh.cuh"
#include "k_sample.cuh"
#include "k_srht.cuh"
#include "k_tpu.cuh"

using namespace tfk;

namespace tfe {

static void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw TfError{TF_CUDA, std::string(what) + ": " + cudaGetErrorString(e)};
}
#define CK(x) cuda_check((x), #x)
static void nccl_check(ncclResult_t r, const char* what);
#define LAUNCH_CHECK(name) cuda_check(cudaGetLastError(), name)
static thread_local int64_t g_launches = 0;
#define COUNT_LAUNCH() (++g_launches)

// Opt a kernel in to `bytes` of dynamic shared memory (monotone per kernel).
// Always, not only above 48 KB: static + dynamic can cross the default limit
// below it.  Serialised: contexts launch from several host threads.
static void smem_optin(const void* func, size_t bytes) {
  static std::mutex mu;
  static std::map<const void*, size_t> have;
  std::lock_guard<std::mutex> lk(mu);
  size_t& h = have[func];
  if (bytes > h) {
    const cudaError_t e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e != cudaSuccess) throw TfError{TF_CUDA, std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e)};
    h = bytes;
  }
}

std::atomic<uint64_t> g_alloc_gen{0};  // bumped by every device (re)allocation

template <class T>
void DBuf<T>::need(size_t count) {
  if (count <= n && p) return;
  g_alloc_gen.fetch_add(1);
  if (p) cudaFree(p);
  p = nullptr;
  n = 0;
  size_t want = std::max<size_t>(count, 1);
  cuda_check(cudaMalloc(&p, want * sizeof(T)), "cudaMalloc");
  n = want;
}

template <class T>
void DBuf<T>::release() {
  if (p) cudaFree(p);
  p = nullptr;
  n = 0;
}

template struct DBuf<double>;
template struct DBuf<int64_t>;
template struct DBuf<int>;
template struct DBuf<uint64_t>;
template struct DBuf<unsigned char>;
template struct DBuf<long long>;
template struct DBuf<unsigned long long>;

static const char* reason_text(int reason) {
  switch (reason) {
    case kReasonZeroResidual: return "zero residual norm; sampling distribution undefined";
    case kReasonNegativeScore: return "negative leverage score";
    case kReasonZeroScoreSum: return "zero score sum; distribution undefined";
    case kReasonCholFail: return "compressed least-squares factorization failed";
    case kReasonRankDeficient: return "reference matrix is rank deficient";
    case kReasonZeroWindow: return "all-zero window; leverage undefined";
    case kReasonSketchStream: return "gaussian sketch stream exhausted";
    default: return "numerical failure";
  }
}

static void raise_from_status(const int st[3]) {
  if (st[0] == 0) return;
  const tf_status code = st[0] == kErrUsage ? TF_USAGE : st[0] == kErrData ? TF_DATA : TF_NUMERICAL;
  throw TfError{code, std::string(reason_text(st[2])) + " (lag " + std::to_string(st[1]) + ")"};
}

// ---------------------------------------------------------------------------
// CholeskyQR2 (shifted CholeskyQR3 on breakdown) solve of one sampled system.
// rows: c gathered rows of width K = p + 1 (gathered order: target first).
// Writes phi (length p) to phi_out, optionally coefs/taus/method at `lag`.
struct SolveOut {
  double* phi;
  double* coefs;
  int64_t coef_off;
  double* taus;
  int* method;
  int lag;
  int* status;
};

struct GramPlan {
  int nblk, npair, nsplit;
  int64_t rps;
};

// leading dimension of the dense tall matrices (Q1, Q2, materialised rows):
// even, so every row starts 16-byte aligned for cp.async
static inline int64_t ldq_of(int K) { return (K + 1) & ~1; }

// split-K plan: ~4 CTAs per SM (3 resident at 70 KB smem each; 3, 6 and 9 per SM measured the same), >= 2 slabs per split
static GramPlan gram_plan(int64_t rows, int K, int sm_count) {
  GramPlan g;
  g.nblk = (K + 63) / 64;
  g.npair = g.nblk * (g.nblk + 1) / 2;
  const int64_t target = 4LL * sm_count;
  int64_t ns = (target + g.npair - 1) / g.npair;
  ns = std::max<int64_t>(1, std::min<int64_t>(ns, (rows + 63) / 64));
  int64_t rps = (rows + ns - 1) / ns;
  rps = (rps + 31) / 32 * 32;
  g.rps = std::max<int64_t>(rps, 32);
  g.nsplit = (int)((rows + g.rps - 1) / g.rps);
  if (g.nsplit < 1) g.nsplit = 1;
  return g;
}

// G (TPU) = Q^T Q for a dense row-major Q (ld even): pipelined DMMA tiles +
// ordered split reduction
static void gram_dense(tf_context* ctx, const double* Q, int64_t ld, int64_t rows, int K, double* G,
                       const int* gate) {
  const GramPlan g = gram_plan(rows, K, ctx->sm_count);
  const size_t smem = gram2_smem_bytes();
  smem_optin((const void*)k_gram_dense_t<kG2Stages>, smem);
  dim3 grid(g.npair, g.nsplit);
  k_gram_dense_t<kG2Stages><<<grid, kGramThreads, smem, ctx->stream>>>(Q, ld, rows, K, g.nblk, g.rps, ctx->sb.W.get(), gate);
  LAUNCH_CHECK("k_gram_dense");
  k_gram_reduce<<<g.npair * 128, 256, 0, ctx->stream>>>(ctx->sb.W.get(), g.npair, g.nsplit, g.nblk, K, G, gate);
  LAUNCH_CHECK("k_gram_reduce");
  g_launches += 2;
}

// G (TPU) = A^T A for loader rows: materialise densely, then gram_dense
template <class L>
static void gram(tf_context* ctx, const L& ld, int64_t rows, int K, double* G, const int* gate) {
  const int64_t lq = ldq_of(K);
  ctx->sb.M.need((size_t)rows * lq);
  dim3 blk(32, 8);
  k_rows_dense<L><<<(unsigned)((rows + 7) / 8), blk, 0, ctx->stream>>>(ld, rows, K, ctx->sb.M.get(), lq);
  LAUNCH_CHECK("k_rows_dense");
  COUNT_LAUNCH();
  gram_dense(ctx, ctx->sb.M.get(), lq, rows, K, G, gate);
}

// Q = A B, B upper-triangular TPU (window-row kernel: row pointers and
// weights staged per CTA, 2-stage cp.async ring; tools/qform_bench.cu)
static WinFwd to_win(const FwdRows& l) { return WinFwd{l.y, l.idx, l.wt, l.off}; }
static WinRev to_win(const RevRows& l) { return WinRev{l.y, l.idx, l.wt, l.base}; }
static WinDense to_win(const DenseRows& l) { return WinDense{l.q, l.ld}; }

template <class L>
static void qform(tf_context* ctx, const L& ld, int64_t rows, int K, const double* B, double* Q,
                  const int* gate) {
  using Wt = decltype(to_win(ld));
  constexpr size_t smem = qform_pipe_smem<2>();
  smem_optin((const void*)k_qform_pipe<Wt, 2, false>, smem);
  dim3 grid((unsigned)((rows + 63) / 64), (unsigned)((K + 63) / 64));
  k_qform_pipe<Wt, 2, false><<<grid, kGramThreads, smem, ctx->stream>>>(to_win(ld), rows, K, B, Q, ldq_of(K),
                                                                       gate);
  LAUNCH_CHECK("k_qform_pipe");
  COUNT_LAUNCH();
}

// blocked multi-launch Cholesky for K > kCholinvMaxK (RD output, no inverse)
static void cholinv_big(tf_context* ctx, const double* G, int K, int pass, int64_t rows, double* RD,
                        const int* gate, int lag, int* status, int force_b) {
  ctx->scratch.need(16);
  ctx->rh_flag.need(8);
  BigChol a;
  a.G = G;
  a.RD = RD;
  a.K = K;
  a.nrows = rows;
  a.pass = pass;
  a.force_b = force_b;
  a.flags = ctx->sb.flags.get();
  a.work = ctx->rh_flag.get() + 4;
  a.tr = ctx->scratch.get() + 8;
  a.gate = gate;
  a.status = status;
  a.lag = lag;
  cudaStream_t st = ctx->stream;
  const int nb = (K + 31) / 32;
  const unsigned cgrid = (unsigned)std::min<int64_t>(148, (tpu_size(K) + 255) / 256);
  for (int attempt = 0; attempt < 2; ++attempt) {
    k_bchol_arm<<<1, 32, 0, st>>>(a, attempt);
    k_bchol_copy<<<cgrid, 256, 0, st>>>(a);
    k_bchol_shift<<<1, 256, 0, st>>>(a);
    g_launches += 3;
    for (int b = 0; b < nb; ++b) {
      k_bchol_diag<<<1, 32, 0, st>>>(a, b);
      ++g_launches;
      if (b + 1 < nb) {
        const int nt = nb - 1 - b;
        k_bchol_panel<<<nt, 64, 0, st>>>(a, b);
        k_bchol_syrk<<<nt * (nt + 1) / 2, 64, 0, st>>>(a, b);
        g_launches += 2;
      }
    }
    if (pass != 0) break;  // only pass A retries with a shift
  }
  k_bchol_finish<<<1, 256, 0, st>>>(a);
  LAUNCH_CHECK("k_bchol");
  COUNT_LAUNCH();
}

static void cholinv(tf_context* ctx, const double* G, int K, int pass, int64_t rows, double* RD,
                    const int* gate, int lag, int* status, int force_b = 0, int invert = 0) {
  if (!cholinv_in_smem(K) && !invert) {
    cholinv_big(ctx, G, K, pass, rows, RD, gate, lag, status, force_b);
    return;
  }
  CholinvArgs a;
  a.G = G;
  a.K = K;
  a.pass = pass;
  a.nrows = rows;
  a.RD = RD;
  a.use_smem = cholinv_in_smem(K) ? 1 : 0;
  a.flags = ctx->sb.flags.get();
  a.gate = gate;
  a.force_b = force_b;
  a.invert = invert;
  a.status = status;
  a.lag = lag;
  const size_t smem = a.use_smem ? cholinv_smem_bytes(K) : 0;
  smem_optin((const void*)k_cholinv, smem);
  k_cholinv<<<1, kCholinvThreads, smem, ctx->stream>>>(a);
  {
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess)
      throw TfError{TF_CUDA, "k_cholinv (K=" + std::to_string(K) + ", smem=" + std::to_string(smem) +
                                 "): " + cudaGetErrorString(e)};
  }
  COUNT_LAUNCH();
}

// X = A Rinv (and X2 = X when non-null) for upper-triangular TPU operands
static void trmm_tpu(tf_context* ctx, const double* A, const double* Rinv, double* X, double* X2, int K,
                     const int* gate) {
  const int nb = (K + 31) / 32;
  k_trmm_tpu<<<nb * (nb + 1) / 2, 64, 0, ctx->stream>>>(A, Rinv, X, X2, K, gate);
  LAUNCH_CHECK("k_trmm_tpu");
  COUNT_LAUNCH();
}

// X = B R^-1 (R in RD format); TPU: B, X upper-triangular K x K; else dense rows x K.
template <bool TPU>
static void trsm_right(tf_context* ctx, const double* B, const double* RD, double* X, int64_t rows,
                       int K, const int* gate) {
  const size_t smem = trsm_smem_bytes(K);
  smem_optin((const void*)k_trsm_right<TPU>, smem);
  const unsigned grid = TPU ? (unsigned)((K + 31) / 32) : (unsigned)((rows + 31) / 32);
  k_trsm_right<TPU><<<grid, kTrsmThreads, smem, ctx->stream>>>(B, RD, X, rows, K, TPU ? K : ldq_of(K), gate);
  LAUNCH_CHECK("k_trsm_right");
  COUNT_LAUNCH();
}

static unsigned tpu_grid(int K) { return (unsigned)std::min<int64_t>(1024, (tpu_size(K) + 255) / 256); }

// split-K workspace for every Gram up to K columns over `rows` rows
static void reserve_gram(tf_context* ctx, int64_t rows, int Kmax) {
  SolveBufs& b = ctx->sb;
  size_t wmax = 0;
  for (int K = 2; K <= Kmax; ++K) {
    const GramPlan g = gram_plan(rows, K, ctx->sm_count);
    wmax = std::max(wmax, (size_t)g.nsplit * g.npair * 4096);
  }
  b.W.need(wmax);
}

// Size every solve buffer for the largest system of a sweep up front so that
// no cudaMalloc/cudaFree (which synchronise) happens between lags.
static void reserve_solve(tf_context* ctx, int64_t c, int Kmax) {
  SolveBufs& b = ctx->sb;
  const size_t tsz = (size_t)tpu_size(std::max(Kmax, 2));
  b.G.need(tsz);
  b.RA.need(tsz);
  b.RB.need(tsz);
  b.RC.need(tsz);
  b.SA.need(tsz);
  b.RI.need(tsz);
  b.SB.need(tsz);
  b.SC.need(tsz);
  b.T.need(tsz);
  b.S0.need(tsz);
  b.S1.need(tsz);
  b.Q1.need((size_t)c * ldq_of(Kmax));
  b.Q2.need((size_t)c * ldq_of(Kmax));
  b.flags.need(4);
  reserve_gram(ctx, c, Kmax);
}

// Preconditioned CholeskyQR solve of one sampled system (forward column
// order, K = p + 1 columns, target last).  `Sprev` (TPU, K - 1) is the
// previous lag's inverse factor (nullptr -> identity preconditioner);
// `Snext` receives this lag's S = R^-1 for the next lag.
// rev = 1: target-first column order (RH lags, RevRows); `rscal` points at the
// squared residual norm that scales the carried preconditioner (LSAR: the
// window's R_{p-1} = scal[0]; RH: the previous lag's sampled estimate), and
// `rest_out` receives this lag's estimate (rev only).
template <class L>
static void solve_rows(tf_context* ctx, const L& ld, int64_t c, int K, const SolveOut& o,
                       const double* Sprev, const double* phi_prev, double* Snext, int rev = 0,
                       const double* rscal = nullptr, double* rest_out = nullptr, bool exact = false) {
  SolveBufs& b = ctx->sb;
  reserve_solve(ctx, c, K);
  int* fl = b.flags.get();
  cudaStream_t st = ctx->stream;
  PhiSArgs pa;
  pa.K = K;
  pa.SA = b.SA.get();
  pa.SB = b.SB.get();
  pa.SC = b.SC.get();
  pa.flags = fl;
  pa.phi = o.phi;
  pa.coefs = o.coefs;
  pa.coef_off = o.coef_off;
  pa.taus = o.taus;
  pa.method = o.method;
  pa.lag = o.lag;
  pa.S_final = Snext ? Snext : b.S0.get();
  pa.rev = rev;
  pa.rest_out = rest_out;
  if (K == 2) {
    gram(ctx, ld, c, K, b.G.get(), nullptr);
    k_solve_k2<<<1, 1, 0, st>>>(b.G.get(), pa);
    LAUNCH_CHECK("k_solve_k2");
    COUNT_LAUNCH();
    return;
  }
  if (Sprev && phi_prev)
    k_precond<<<tpu_grid(K), 256, 0, st>>>(Sprev, phi_prev, rscal ? rscal : ctx->scal.get(),
                                           b.T.get(), K);
  else
    k_tpu_identity<<<tpu_grid(K), 256, 0, st>>>(b.T.get(), K);
  LAUNCH_CHECK("k_precond");
  COUNT_LAUNCH();
  double* Sfin = pa.S_final;
  const int64_t lq = ldq_of(K);
  const int forceb = (Sprev && phi_prev) ? 0 : 1;
  if (exact) {
    // exact S (RH generalized leverage): the Cholesky kernel returns R^-1 and
    // S = T R_A^-1 [R_B^-1 [R_C^-1]] is formed by triangular products
    qform(ctx, ld, c, K, b.T.get(), b.Q1.get(), nullptr);
    gram_dense(ctx, b.Q1.get(), lq, c, K, b.G.get(), nullptr);
    cholinv(ctx, b.G.get(), K, 0, c, b.RA.get(), nullptr, o.lag, o.status, forceb, 1);
    trmm_tpu(ctx, b.T.get(), b.RA.get(), b.SA.get(), Sfin, K, nullptr);
    DenseRows q1{b.Q1.get(), lq}, q2{b.Q2.get(), lq};
    qform(ctx, q1, c, K, b.RA.get(), b.Q2.get(), fl + 2);
    gram_dense(ctx, b.Q2.get(), lq, c, K, b.G.get(), fl + 2);
    cholinv(ctx, b.G.get(), K, 1, c, b.RB.get(), fl + 2, o.lag, o.status, 0, 1);
    trmm_tpu(ctx, b.SA.get(), b.RB.get(), b.SB.get(), Sfin, K, fl + 2);
    qform(ctx, q2, c, K, b.RB.get(), b.Q1.get(), fl + 0);
    gram_dense(ctx, b.Q1.get(), lq, c, K, b.G.get(), fl + 0);
    cholinv(ctx, b.G.get(), K, 2, c, b.RC.get(), fl + 0, o.lag, o.status, 0, 1);
    trmm_tpu(ctx, b.SB.get(), b.RC.get(), b.SC.get(), Sfin, K, fl + 0);
    k_phi_S<<<1, 256, 0, st>>>(pa);
    LAUNCH_CHECK("k_phi_S");
    COUNT_LAUNCH();
    return;
  }
  // fast path (sweep lags, standalone solves): factors only; phi by O(K^2)
  // substitutions; the next lag's preconditioner S ~ T R^-1 to first order
  qform(ctx, ld, c, K, b.T.get(), b.Q1.get(), nullptr);
  gram_dense(ctx, b.Q1.get(), lq, c, K, b.G.get(), nullptr);
  cholinv(ctx, b.G.get(), K, 0, c, b.RA.get(), nullptr, o.lag, o.status, forceb, 0);
  const unsigned npair = (unsigned)(((K + 31) / 32) * ((K + 31) / 32 + 1) / 2);
  if (Snext) {
    k_rinv_first_order<<<npair, 64, 0, st>>>(b.RA.get(), b.RI.get(), K, nullptr);
    COUNT_LAUNCH();
    trmm_tpu(ctx, b.T.get(), b.RI.get(), b.SA.get(), Snext, K, nullptr);
  }
  // pass B (gated): Q2 = Q1 R_A^-1 by blocked substitution
  trsm_right<false>(ctx, b.Q1.get(), b.RA.get(), b.Q2.get(), c, K, fl + 2);
  gram_dense(ctx, b.Q2.get(), lq, c, K, b.G.get(), fl + 2);
  cholinv(ctx, b.G.get(), K, 1, c, b.RB.get(), fl + 2, o.lag, o.status);
  if (Snext) {
    k_rinv_first_order<<<npair, 64, 0, st>>>(b.RB.get(), b.RI.get(), K, fl + 2);
    COUNT_LAUNCH();
    trmm_tpu(ctx, b.SA.get(), b.RI.get(), b.SB.get(), Snext, K, fl + 2);
  }
  // pass C (gated: pass A shifted): Q1 = Q2 R_B^-1
  trsm_right<false>(ctx, b.Q2.get(), b.RB.get(), b.Q1.get(), c, K, fl + 0);
  gram_dense(ctx, b.Q1.get(), lq, c, K, b.G.get(), fl + 0);
  cholinv(ctx, b.G.get(), K, 2, c, b.RC.get(), fl + 0, o.lag, o.status);
  if (Snext) {
    k_rinv_first_order<<<npair, 64, 0, st>>>(b.RC.get(), b.RI.get(), K, fl + 0);
    COUNT_LAUNCH();
    trmm_tpu(ctx, b.SB.get(), b.RI.get(), b.SC.get(), Snext, K, fl + 0);
  }
  PhiSolveArgs ps;
  ps.K = K;
  ps.T = b.T.get();
  ps.RA = b.RA.get();
  ps.RB = b.RB.get();
  ps.RC = b.RC.get();
  ps.flags = fl;
  ps.rev = rev;
  ps.phi = o.phi;
  ps.coefs = o.coefs;
  ps.coef_off = o.coef_off;
  ps.taus = o.taus;
  ps.method = o.method;
  ps.lag = o.lag;
  ps.rest_out = rest_out;
  k_phi_solve<<<1, kPhiThreads, (size_t)(2 * K + 32) * sizeof(double), st>>>(ps);
  LAUNCH_CHECK("k_phi_solve");
  COUNT_LAUNCH();
  // rank-deficient / breakdown systems: the reference's minimum-norm answer
  // (gated on the shift flag inside the kernel; small systems only)
  if (c * (int64_t)(K - 1) <= kMinNormCap && K - 1 <= 64 && c <= 4096) {
    const size_t smem = sizeof(double) * ((size_t)c * (K - 1) + c + 2 * (size_t)(K - 1) * (K - 1));
    smem_optin((const void*)k_minnorm<L>, smem);
    k_minnorm<L><<<1, kMinNormThreads, smem, st>>>(ld, c, K, rev, fl, o.phi, o.coefs, o.coef_off, o.taus,
                                                   o.method, o.lag, o.status);
    LAUNCH_CHECK("k_minnorm");
    COUNT_LAUNCH();
  }
}

// ---------------------------------------------------------------------------
// The reference's rank-revealing solve of a sampled lag system at every K
// (toeplitz.cpp:57-85; k_exact.cuh): double-double Gram -> pivoted Cholesky
// (= CPQR) -> phi by back-substitution, or the minimum-norm SVD answer when
// the rank rule finds rank < p.  rev = 1: target-first column order (RH).
constexpr int kExactMaxP = 640;  // the SVD block pair of a 16-CTA cluster fits shared memory up to here

// launch shape of k_svd_minnorm for lag order p: nct CTAs (nblk = 2 nct
// blocks) cover the worst case ncol = p; bw = the block width the shared
// memory is sized for (>= p / nblk, up to 32 = a warp per pair, within the
// opt-in limit) -- the kernel picks its block count from the actual ncol
static void svd_plan(int p, int smem_max, int& nct, int& nblk, int& bw) {
  nct = std::min(kSvdMaxCta, std::max(1, (p + 31) / 32));
  nblk = 2 * nct;
  const int fit = (int)((size_t)(smem_max - 2048) / svd_smem_bytes(p, 1));  // static shared memory: 1 KB
  bw = std::max((p + nblk - 1) / nblk, std::min(kSvdThreads / 32, fit));
}

// INT8 tensor-core Gram (k_i8gram.cuh) or the double-double CUDA-core one
// (k_gram_dd): both produce the same (hi, lo) Gram to ~1e-27 relative; the
// tensor-core path pays a fixed slicing cost, so it is taken above a work
// threshold (c K^2, measured crossover on B200) and while the int32 products
// are exact (c <= kI8MaxRows).
constexpr int kI8MaxNbs = 6;  // K <= 768
static bool use_i8_gram(const tf_context* ctx, int64_t c, int K) {
  if (ctx->gram_mode == 1 || c > kI8MaxRows || K > kI8MaxNbs * kI8Tile) return false;
  return ctx->gram_mode == 2 || (double)c * K * K >= kI8MinWork;
}

// K splits of the INT8 GEMM: only when the tiles fill less than half the SMs
// (K <= 128: 31 tiles), then as many as fill one wave (>= 64 K steps each);
// more tiles than that gained nothing measurable (the partial tiles' epilogue
// and the combine's extra reads eat the wave-quantisation gain)
static int i8_ksplit(int ntiles, int64_t nk, int sms) {
  if (2 * ntiles > sms) return 1;
  int ks = std::max(1, sms / ntiles);
  while (ks > 1 && nk / ks < 64) --ks;
  return std::min(ks, 8);
}

static void i8_tables(tf_context* ctx) {
  SolveBufs& b = ctx->sb;
  if (!b.i8_ntiles.empty()) return;
  std::vector<int> tl, tof;
  b.i8_tile_off.assign(kI8MaxNbs + 1, 0);
  b.i8_tof_off.assign(kI8MaxNbs + 1, 0);
  b.i8_ntiles.assign(kI8MaxNbs + 1, 0);
  for (int nbs = 1; nbs <= kI8MaxNbs; ++nbs) {
    const int nbt = kI8S * nbs;
    b.i8_tile_off[nbs] = (int)tl.size() / 2;
    b.i8_tof_off[nbs] = (int)tof.size();
    const size_t t0 = tof.size();
    tof.resize(t0 + (size_t)nbt * nbt, -1);
    // tiles (I, m) of 128 x 256 (blocks I and 2m, 2m + 1), kept when either
    // half holds a needed (I <= J, s + u <= S - 1) block pair; launch order:
    // B x B blocks of tiles, so that the ~148 tiles in flight read few
    // distinct digit panels (each 128 B x c rows) and stream them from L2
    // together instead of re-reading them from DRAM
    static const int B = std::getenv("TF_I8_BLOCK") ? std::max(1, std::atoi(std::getenv("TF_I8_BLOCK"))) : 8;
    auto need = [&](int I, int J) { return I <= J && I / nbs + J / nbs <= kI8S - 1; };
    std::vector<std::pair<int, int>> pairs;
    for (int I = 0; I < nbt; ++I)
      for (int m = I / 2; m < nbt / 2; ++m)
        if (need(I, 2 * m) || need(I, 2 * m + 1)) pairs.emplace_back(I, m);
    std::stable_sort(pairs.begin(), pairs.end(), [](const std::pair<int, int>& x, const std::pair<int, int>& y) {
      const int bx = x.first / B, by = y.first / B, cx = x.second / B, cy = y.second / B;
      return bx != by ? bx < by : cx < cy;
    });
    int cnt = 0;
    for (const auto& im : pairs) {
      for (int h = 0; h < 2; ++h)
        if (need(im.first, 2 * im.second + h)) tof[t0 + (size_t)im.first * nbt + 2 * im.second + h] = 2 * cnt + h;
      tl.push_back(im.first);
      tl.push_back(im.second);
      ++cnt;
    }
    b.i8_ntiles[nbs] = cnt;
  }
  b.i8tiles.need(tl.size());
  b.i8tof.need(tof.size());
  CK(cudaMemcpy(b.i8tiles.get(), tl.data(), tl.size() * sizeof(int), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(b.i8tof.get(), tof.data(), tof.size() * sizeof(int), cudaMemcpyHostToDevice));
}

static void reserve_exact(tf_context* ctx, int64_t c, int Kmax) {
  SolveBufs& b = ctx->sb;
  size_t wmax = 0;
  int ki8 = 0;
  for (int K = 2; K <= Kmax; ++K) {
    if (use_i8_gram(ctx, c, K)) {
      ki8 = K;
      continue;
    }
    const GramDDPlan g = gram_dd_plan(c, K, ctx->sm_count);
    wmax = std::max(wmax, (size_t)g.npair * g.nsplit * 8192);
  }
  const size_t KK = (size_t)Kmax * Kmax;
  if (wmax) b.Wdd.need(wmax);
  if (ki8) {
    i8_tables(ctx);
    const int nbs = (ki8 + kI8Tile - 1) / kI8Tile;
    const int64_t cpad = (c + kI8Tile - 1) / kI8Tile * kI8Tile;
    b.i8D.need((size_t)kI8S * nbs * kI8Tile * cpad);
    b.i8E.need((size_t)nbs * kI8Tile);
    {
      size_t mx = 0;  // the largest (tiles x splits) of any block count up to nbs
      for (int nb = 1; nb <= nbs; ++nb)
        mx = std::max(mx, (size_t)b.i8_ntiles[nb] * i8_ksplit(b.i8_ntiles[nb], (c + kI8Tile - 1) / kI8Tile, ctx->sm_count));
      b.i8P.need(mx * kI8Tile * kI8N);
    }
  }
  b.Gh.need(KK);
  b.Gl.need(KK);
  b.Rh.need(KK);
  b.Rl.need(KK);
  b.Nsv.need((size_t)Kmax * Kmax);
  b.sig.need(Kmax);
  b.xpart.need((size_t)2 * kSvdMaxCta * Kmax);
  b.tolv.need(2);
  b.Dd.need((size_t)4 * Kmax);
  b.cn.need(Kmax);
  b.cnp.need((size_t)((c + kCnRows - 1) / kCnRows) * Kmax);
  b.perm.need(Kmax);
  b.svdf.need(72);  // [0] deficient, [1] rank, [2..65] sweep flags, [66] nonzero rows of R'
}

// rows_dev (nullable): the device-side row count (a shard's draws, <= c);
// sharded: the Gram partials are allgathered over ctx->comm and summed in rank
// order, so every rank factors the same double-double Gram.
template <class L>
// ybits (nullable, FwdRows only): max |y| of the resident series (k_absmax_bits): the
// INT8 Gram takes its digit exponents from max |w| * max |y| instead of a column-max pass
static void solve_exact(tf_context* ctx, const L& ld, int64_t c, int K, int rev, const ExactOut& o,
                        const long long* rows_dev = nullptr, bool sharded = false,
                        const unsigned long long* ybits = nullptr) {
  SolveBufs& b = ctx->sb;
  cudaStream_t st = ctx->stream;
  const int p = K - 1;
  if (p > kExactMaxP) throw TfError{TF_USAGE, "lag order above " + std::to_string(kExactMaxP) + " (rank-revealing solve)"};
  const int64_t KK = (int64_t)K * K;
  double* gh = sharded ? b.Gloc.get() : b.Gh.get();
  double* gl = sharded ? b.Gloc.get() + KK : b.Gl.get();
  const unsigned ns = (unsigned)((c + kCnRows - 1) / kCnRows);
  if (use_i8_gram(ctx, c, K)) {
    const int nbs = (K + kI8Tile - 1) / kI8Tile, Kp = nbs * kI8Tile;
    const int64_t nk = (c + kI8Tile - 1) / kI8Tile;
    if constexpr (std::is_same<L, FwdRows>::value) {
      if (ybits) {
        k_i8_exp_fwd<<<1, 1024, 0, st>>>(ld.wt, c, rows_dev, ybits, K, b.i8E.get());
      } else {
        k_i8_colmax_part<L><<<dim3((unsigned)((K + 63) / 64), ns), 256, 0, st>>>(ld, c, K, rows_dev, b.cnp.get());
        k_i8_colmax_fin<<<(unsigned)((K + 127) / 128), 128, 0, st>>>(b.cnp.get(), (int)ns, K, b.i8E.get());
      }
    } else {
      k_i8_colmax_part<L><<<dim3((unsigned)((K + 63) / 64), ns), 256, 0, st>>>(ld, c, K, rows_dev, b.cnp.get());
      k_i8_colmax_fin<<<(unsigned)((K + 127) / 128), 128, 0, st>>>(b.cnp.get(), (int)ns, K, b.i8E.get());
    }
    k_i8_slice<L><<<dim3((unsigned)nk, (unsigned)(Kp / 32)), 256, 0, st>>>(ld, c, K, Kp, nk, rows_dev, b.i8E.get(),
                                                                           (int8_t*)b.i8D.get());
    LAUNCH_CHECK("k_i8_slice");
    smem_optin((const void*)k_i8_gemm, kI8Smem);
    const int ntiles = b.i8_ntiles[nbs], ks = i8_ksplit(ntiles, nk, ctx->sm_count);
    k_i8_gemm<<<(unsigned)(ntiles * ks), kI8Threads, kI8Smem, st>>>(
        (const int8_t*)b.i8D.get(), nk, reinterpret_cast<const int2*>(b.i8tiles.get()) + b.i8_tile_off[nbs],
        b.i8P.get(), ntiles, ks);
    LAUNCH_CHECK("k_i8_gemm");
    k_i8_combine<<<(unsigned)((KK + 255) / 256), 256, 0, st>>>(b.i8P.get(), b.i8tof.get() + b.i8_tof_off[nbs],
                                                              kI8S * nbs, K, Kp, b.i8E.get(), gh, gl, ntiles, ks);
    LAUNCH_CHECK("k_i8_combine");
    g_launches += 5;
  } else {
    const GramDDPlan g = gram_dd_plan(c, K, ctx->sm_count);
    // column sums of squares: the accumulation bias of each Gram element
    k_colnorm2_part<L><<<dim3((unsigned)((K + 63) / 64), ns), 256, 0, st>>>(ld, c, K, rows_dev, b.cnp.get());
    k_colnorm2_sum<<<(unsigned)((K + 127) / 128), 128, 0, st>>>(b.cnp.get(), (int)ns, K, b.cn.get());
    LAUNCH_CHECK("k_colnorm2");
    k_gram_dd<L><<<dim3((unsigned)g.npair, (unsigned)g.nsplit), kDDThreads, 0, st>>>(ld, c, K, g.nblk, g.rps, g.nsplit,
                                                                                    b.Wdd.get(), rows_dev, b.cn.get());
    LAUNCH_CHECK("k_gram_dd");
    k_gram_dd_reduce<<<(unsigned)(((int64_t)g.npair * 4096 + 255) / 256), 256, 0, st>>>(
        b.Wdd.get(), g.npair, g.nsplit, g.nblk, K, gh, gl, nullptr);
    LAUNCH_CHECK("k_gram_dd_reduce");
    g_launches += 4;
  }
  if (sharded) {
    nccl_check(ncclAllGather(b.Gloc.get(), b.Gg.get(), (size_t)(2 * KK), ncclDouble, ctx->comm, st), "ncclAllGather");
    k_dd_sum_ranks<<<(unsigned)((KK + 255) / 256), 256, 0, st>>>(b.Gg.get(), ctx->nc_world, KK, b.Gh.get(), b.Gl.get());
    LAUNCH_CHECK("k_dd_sum_ranks");
    g_launches += 1;
  }
  PcholArgs pa{};
  pa.Gh = b.Gh.get();
  pa.Gl = b.Gl.get();
  pa.K = K;
  pa.rev = rev;
  pa.rows = c;
  pa.Rh = b.Rh.get();
  pa.Rl = b.Rl.get();
  pa.N = b.Nsv.get();
  pa.perm = b.perm.get();
  pa.svd = b.svdf.get();
  pa.tol = b.tolv.get();
  pa.o = o;
  pa.gate = nullptr;
  pa.Dh = b.Dd.get();
  pa.Dl = b.Dd.get() + 2 * K;
  {
    static const int scheme = std::getenv("TF_PCHOL") ? std::atoi(std::getenv("TF_PCHOL")) : 1;  // dev switch: 0 = at most 8 CTAs
    const int pc = pchol_ctas(K, scheme);
    if (pc > 8) {
      static std::once_flag once;
      std::call_once(once, [] {
        CK(cudaFuncSetAttribute((const void*)k_pchol_dd, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
      });
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)pc);
    cfg.blockDim = dim3(kPcThreads);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = (unsigned)pc;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    CK(cudaLaunchKernelEx(&cfg, k_pchol_dd, pa));
  }
  int nct, nblk, bw;
  svd_plan(p, ctx->smem_optin_max, nct, nblk, bw);
  SvdArgs sa{};
  sa.N = b.Nsv.get();
  sa.sig = b.sig.get();
  sa.xpart = b.xpart.get();
  sa.perm = b.perm.get();
  sa.svd = b.svdf.get();
  sa.tol = b.tolv.get();
  sa.p = p;
  sa.nblk = nblk;
  sa.bw = bw;
  sa.rev = rev;
  sa.o = o;
  const size_t smem = svd_smem_bytes(p, bw);
  {
    static std::mutex mu;
    static bool attr = false;
    std::lock_guard<std::mutex> lk(mu);
    if (!attr) {
      CK(cudaFuncSetAttribute((const void*)k_svd_minnorm, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
      attr = true;
    }
  }
  smem_optin((const void*)k_svd_minnorm, smem);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)nct);
  cfg.blockDim = dim3(kSvdThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = (unsigned)nct;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  CK(cudaLaunchKernelEx(&cfg, k_svd_minnorm, sa));
  g_launches += 2;
}

// ---------------------------------------------------------------------------

constexpr int kPassPstMinQ = 1;  // sweeps: tensor-core persistent pass for every lag q >= 1

// FFT pass (k_fft.cuh) for the lags where the direct FIR is fp64-bound; the
// crossover (lag kFftMinQ) is measured (the FFT pass is faster
// from lag 61 on at C4).  A sweep uses it only when enough lags (kFftMinLags)
// follow the crossover to pay for the once-per-sweep series spectra (about
// seven lag passes).
constexpr int kFftMinQ = 64;
constexpr int kFftMinLags = 32;

static bool fft_sweep(const tf_context* ctx, int p_bar) {
  if (ctx->pass_mode == 1 || p_bar > kFftD) return false;
  return ctx->pass_mode == 2 || p_bar >= ctx->fft_minq + ctx->fft_minlags;
}
static bool fft_lag(const tf_context* ctx, int p_bar, int q) {
  return q >= 1 && fft_sweep(ctx, p_bar) && (ctx->pass_mode == 2 || q >= ctx->fft_minq);
}

// buffers of the FFT pass (before any capture): spectra of ceil(w / 6144)
// superblocks, the filter spectrum, the twiddle tables (once per context)
static void reserve_fft(tf_context* ctx, int64_t w) {
  const int64_t nsb = (w + kFftSB - 1) / kFftSB;
  ctx->fftZ.need((size_t)nsb * kFftN);
  ctx->fftH.need(kFftN);
  if (!ctx->fftTw.get()) {
    ctx->fftTw.need(kFftTw);
    std::vector<double2> tw(kFftTw);
    const long double pi = 3.141592653589793238462643383279502884L;
    for (int e = 0; e < 256; ++e) {
      const long double a256 = -2.0L * pi * e / 256.0L, a4096 = -2.0L * pi * e / 4096.0L;
      tw[e] = make_double2((double)cosl(a256), (double)sinl(a256));
      tw[256 + e] = make_double2((double)cosl(a4096), (double)sinl(a4096));
    }
    CK(cudaMemcpy(ctx->fftTw.get(), tw.data(), kFftTw * sizeof(double2), cudaMemcpyHostToDevice));
    // double-double W_4096^e for the spectra (k_fft_series_dd, k_fft_taps_dd):
    // hi = the rounded long double value, lo = the long double remainder
    std::vector<double2> th(kFftN), tl(kFftN);
    for (int e = 0; e < kFftN; ++e) {
      const long double a = -2.0L * pi * e / (long double)kFftN;
      const long double c = cosl(a), s = sinl(a);
      th[e] = make_double2((double)c, (double)s);
      tl[e] = make_double2((double)(c - (long double)th[e].x), (double)(s - (long double)th[e].y));
    }
    ctx->fftTwH.need(kFftN);
    ctx->fftTwL.need(kFftN);
    CK(cudaMemcpy(ctx->fftTwH.get(), th.data(), kFftN * sizeof(double2), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(ctx->fftTwL.get(), tl.data(), kFftN * sizeof(double2), cudaMemcpyHostToDevice));
  }
  smem_optin((const void*)k_fft_series_dd, fft_dd_smem_bytes());
  smem_optin((const void*)k_lsar_pass_fft<0>, fft_smem_bytes());
  smem_optin((const void*)k_lsar_pass_fft<1>, fft_smem_bytes());
  smem_optin((const void*)k_lsar_pass_fft<2>, fft_smem_bytes());
  smem_optin((const void*)k_lsar_pass_fft<3>, fft_smem_bytes());
  smem_optin((const void*)k_lsar_pass_fft<4>, fft_smem_bytes());
  smem_optin((const void*)k_lsar_pass_fft<4, 1>, fft_smem_bytes(fft_tw_entries<1>()));
  smem_optin((const void*)k_lsar_pass_fft_r, fft_smem_bytes(fft_tw_entries<1>()));
  CK(cudaFuncSetAttribute((const void*)k_lsar_pass_fft_r, cudaFuncAttributePreferredSharedMemoryCarveout, 70));
  // two CTAs of 78 KB: the 164 KB shared-memory carve-out (70 % of 228 KB rounds up to it; 72 % gave 196 KB) leaves ~92 KB of L1, which keeps H (64 KB) resident
  CK(cudaFuncSetAttribute((const void*)k_lsar_pass_fft<4, 1>, cudaFuncAttributePreferredSharedMemoryCarveout, 70));

}

static int fft_grid(const tf_context* ctx, int64_t nsb) {
  return (int)std::min<int64_t>(nsb, 2 * (int64_t)ctx->sm_count);
}

// spectra of the resident series (y[0 .. n)) for a window of w rows
static void launch_fft_series(tf_context* ctx, int64_t w) {
  const int64_t nsb = (w + kFftSB - 1) / kFftSB;
  k_fft_series_dd<<<(int)std::min<int64_t>(nsb, ctx->sm_count), kFftT, fft_dd_smem_bytes(), ctx->stream>>>(
      ctx->y.get(), ctx->n, nsb, ctx->fftZ.get(), ctx->fftTwH.get(), ctx->fftTwL.get());
  LAUNCH_CHECK("k_fft_series_dd");
  COUNT_LAUNCH();
}

// Deferred folding plan of one sweep (k_fft.cuh, kFftSlots): q0 = the first
// FFT lag, K groups; residual r_j (j >= q0 - 1) lives in slot (j - q0 + 1) mod M,
// M = K + 1 slots (slot 0 = ctx->r, where the direct pass of lag q0 - 1 left
// it): r_q's slot is never one of the K pending residuals, so the pass may
// write r_q before it folds.  K = 1: the classic state (s_q, r_q in place every
// lag, M = 1).
struct FoldPlan {
  int K = 1, M = 1, q0 = 0;
  int64_t grid = 1;  // the FFT pass's grid (superblock groups depend on it)
  double* slot[kFftSlots + 1] = {};
  double* of(int lag) const { return slot[((lag - q0 + 1) % M + M) % M]; }
  // last lag <= at at which group g folded (q0 - 1: never, the state the direct pass left)
  int last_fold(int g, int at) const {
    if (at < q0 + g) return q0 - 1;
    return q0 + g + ((at - q0 - g) / K) * K;
  }
};

static FoldPlan fold_plan(tf_context* ctx, int p_bar, int64_t w) {
  FoldPlan f;
  int q0 = 1;
  while (q0 <= p_bar && !fft_lag(ctx, p_bar, q0)) ++q0;
  f.q0 = q0;
  // groups beyond the FFT lags' count buy nothing
  f.K = std::max(1, std::min(ctx->fft_slots, p_bar - q0 + 1));
  f.grid = fft_grid(ctx, (w + kFftSB - 1) / kFftSB);
  f.M = f.K > 1 ? f.K + 1 : 1;
  f.slot[0] = ctx->r.get();
  for (int k = 1; k < f.M; ++k) {
    ctx->fft_rslot[k - 1].need(w);
    f.slot[k] = ctx->fft_rslot[k - 1].get();
  }
  return f;
}

// the row-mass state a draw at lag p sees (the pass of lag p - 1 is done); K = 0
// when that pass was not an FFT pass or K = 1 (the classic s, r)
static PendState pend_state(const FoldPlan& f, int p, const double* Rhist) {
  PendState ps{};
  ps.K = 0;
  if (f.K <= 1 || p - 1 < f.q0) return ps;
  ps.K = f.K;
  ps.sbrows = kFftSB;
  ps.sbgrid = f.grid;
  ps.navail = std::min(f.K, p - f.q0 + 1);
  for (int k = 0; k < ps.navail; ++k) ps.pend[k] = f.of(p - ps.navail + k);
  ps.Rp = Rhist + (p - ps.navail);
  for (int g = 0; g < f.K; ++g) ps.npg[g] = p - f.last_fold(g, p - 1);
  return ps;
}

static FftPassArgs fft_pass_args(tf_context* ctx, int q, int64_t w, const double* Rprev, const FoldPlan& f) {
  FftPassArgs a{};
  a.Z = ctx->fftZ.get();
  a.H = ctx->fftH.get();
  a.tw = ctx->fftTw.get();
  a.w = w;
  a.s = ctx->s.get();
  a.K = f.K;
  if (f.K <= 1) {  // classic: s_q = s_{q-1} + r_{q-1}^2 / R_{q-1}, r_q over r_{q-1}
    a.fold = 0;
    a.npend = 1;
    a.pend[0] = ctx->r.get();
    a.Rp = Rprev;
    a.rout = ctx->r.get();
  } else {
    a.fold = (q - f.q0) % f.K;
    a.npend = q - f.last_fold(a.fold, q - 1);
    for (int k = 0; k < a.npend; ++k) a.pend[k] = f.of(q - a.npend + k);
    a.Rp = ctx->Rhist.get() + (q - a.npend);
    a.rout = f.of(q);
  }
  a.chunkA = ctx->chunkA.get();
  a.chunkB = ctx->chunkB.get();
  a.tileA = ctx->tileA.get();
  a.tileB = ctx->tileB.get();
  a.ggrid = (int)f.grid;
  return a;
}

// the scores of lag q (k_fft_fold) on the side stream: everything it reads is there once the draws
// of lag q are done; the caller orders it after them and joins it before the pass of lag q
static void launch_fft_fold(tf_context* ctx, int q, int64_t w, const double* Rprev, const FoldPlan& f,
                            cudaStream_t stream) {
  FftPassArgs a = fft_pass_args(ctx, q, w, Rprev, f);
  const int64_t nsb = (w + kFftSB - 1) / kFftSB;
  k_fft_fold<<<(unsigned)((nsb + kFoldSB - 1) / kFoldSB), kFftT, 0, stream>>>(a);
  LAUNCH_CHECK("k_fft_fold");
  COUNT_LAUNCH();
}

// split: the scores were k_fft_fold's (launch_fft_fold); the pass writes r_q and the B sums only
static void launch_pass_fft(tf_context* ctx, int q, int64_t w, const double* phi, const double* Rprev,
                            const FoldPlan& f, bool split = false) {
  k_fft_taps_dd<<<kFftN * kTapSplit / 256, 256, 0, ctx->stream>>>(phi, q, ctx->fftH.get(), ctx->fftTwH.get(),
                                                                   ctx->fftTwL.get());
  FftPassArgs a = fft_pass_args(ctx, q, w, Rprev, f);
  a.split = split ? 1 : 0;
  const int64_t nsb = (w + kFftSB - 1) / kFftSB;
  // prefetch variant (dev switch TF_FFT_PF, measured in profiles/r02_fft_prefetch.txt): 4 (state of
  // this superblock and spectrum of the next to L2, the spectrum through shared memory by TMA) is the fastest
  static const int pf = std::getenv("TF_FFT_PF") ? std::atoi(std::getenv("TF_FFT_PF")) : 4;
  // twiddles (dev switch TF_FFT_TW): 1 = powers of one table entry per stage formed in registers
  static const int twm = std::getenv("TF_FFT_TW") ? std::atoi(std::getenv("TF_FFT_TW")) : 1;
  // split: the fused kernel with its score phase skipped.  Dev switch TF_FFT_RPF=1: k_lsar_pass_fft_r, the
  // next spectrum prefetched into registers instead of staged through shared memory by TMA -- measured
  // slower at C4 (4.69 vs 4.54 s per sweep: profiles/r02_fft_prefetch.txt), so off
  static const int rpf = std::getenv("TF_FFT_RPF") ? std::atoi(std::getenv("TF_FFT_RPF")) : 0;
  if (split && pf == 4 && twm == 1 && rpf)
    k_lsar_pass_fft_r<<<fft_grid(ctx, nsb), kFftT, fft_smem_bytes(fft_tw_entries<1>()), ctx->stream>>>(a);
  else if (pf == 4 && twm == 1)
    k_lsar_pass_fft<4, 1><<<fft_grid(ctx, nsb), kFftT, fft_smem_bytes(fft_tw_entries<1>()), ctx->stream>>>(a);
  else if (pf == 0) k_lsar_pass_fft<0><<<fft_grid(ctx, nsb), kFftT, fft_smem_bytes(), ctx->stream>>>(a);
  else if (pf == 1) k_lsar_pass_fft<1><<<fft_grid(ctx, nsb), kFftT, fft_smem_bytes(), ctx->stream>>>(a);
  else if (pf == 3) k_lsar_pass_fft<3><<<fft_grid(ctx, nsb), kFftT, fft_smem_bytes(), ctx->stream>>>(a);
  else if (pf == 4) k_lsar_pass_fft<4><<<fft_grid(ctx, nsb), kFftT, fft_smem_bytes(), ctx->stream>>>(a);
  else k_lsar_pass_fft<2><<<fft_grid(ctx, nsb), kFftT, fft_smem_bytes(), ctx->stream>>>(a);
  LAUNCH_CHECK("k_lsar_pass_fft");
  g_launches += 2;
}

// after the last pass (lag p_bar) of a deferred sweep: s_{p_bar} (every group's
// pending residuals but r_{p_bar} folded) and r_{p_bar} into ctx->s / ctx->r
__global__ void k_fold_all(double* __restrict__ s, double* __restrict__ r, int64_t w, PendState ps) {
  const int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= w) return;
  const double rl = ps.pend[ps.navail - 1][row];
  ps.navail -= 1;  // r_{p_bar} stays unfolded
  const int64_t sb = row / ps.sbrows;
  const int g = (int)((sb + sb / ps.sbgrid) % ps.K);
  if (g == 0) ps.npg[0] -= 1;
  else if (g == 1) ps.npg[1] -= 1;
  else if (g == 2) ps.npg[2] -= 1;
  else ps.npg[3] -= 1;
  s[row] = pend_mass(ps, s, row);
  r[row] = rl;
}

static void finish_fold(tf_context* ctx, const FoldPlan& f, int p_bar, int64_t w) {
  const PendState ps = pend_state(f, p_bar + 1, ctx->Rhist.get());
  if (ps.K <= 1) return;
  k_fold_all<<<(unsigned)((w + 255) / 256), 256, 0, ctx->stream>>>(ctx->s.get(), ctx->r.get(), w, ps);
  LAUNCH_CHECK("k_fold_all");
  COUNT_LAUNCH();
}

// max |y| over the window's series values (y[0 .. rows)) into ctx->ymax (bit pattern)
static void launch_absmax(tf_context* ctx, int64_t rows, const unsigned long long* dst) {
  CK(cudaMemsetAsync((void*)dst, 0, sizeof(unsigned long long), ctx->stream));
  k_absmax_bits<<<2 * ctx->sm_count, 512, 0, ctx->stream>>>(ctx->y.get(), rows, (unsigned long long*)dst);
  LAUNCH_CHECK("k_absmax_bits");
  COUNT_LAUNCH();
}

static void launch_pass(tf_context* ctx, int q, int64_t w, const double* phi, const double* Rprev,
                        bool exact_order = false) {
  PassArgs a{};
  a.y = ctx->y.get();
  a.w = w;
  a.q = q;
  a.phi = phi;
  a.s = ctx->s.get();
  a.r = ctx->r.get();
  a.Rprev = Rprev;
  a.chunkA = ctx->chunkA.get();
  a.chunkB = ctx->chunkB.get();
  a.tileA = ctx->tileA.get();
  a.tileB = ctx->tileB.get();
  a.ylen = ctx->n + 64;
  const int64_t ntile = (w + kPassTile - 1) / kPassTile;
  if (!exact_order && q >= kPassPstMinQ) {
    const size_t smem = PassLayout(q).bytes();
    smem_optin((const void*)k_lsar_pass_pst<0>, smem);
    static std::mutex mu;  // contexts launch from several host threads
    static std::map<size_t, int> occ_of;
    int occ;
    {
      std::lock_guard<std::mutex> lk(mu);
      auto it = occ_of.find(smem);
      if (it == occ_of.end()) {
        int o = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, k_lsar_pass_pst<0>, kPassThreads, smem));
        it = occ_of.emplace(smem, o).first;
      }
      occ = it->second;
    }
    const int64_t grid = std::min<int64_t>(ntile, (int64_t)std::max(occ, 1) * ctx->sm_count);
    k_lsar_pass_pst<0><<<(unsigned)grid, kPassThreads, smem, ctx->stream>>>(a);
    LAUNCH_CHECK("k_lsar_pass_pst");
    COUNT_LAUNCH();
    return;
  }
  const size_t smem = pass_smem_bytes(q);
  smem_optin((const void*)k_lsar_pass, smem);
  k_lsar_pass<<<(unsigned)ntile, kPassThreads, smem, ctx->stream>>>(a);
  LAUNCH_CHECK("k_lsar_pass");
  COUNT_LAUNCH();
}

static void launch_scan(tf_context* ctx, int64_t ntile, int lag, int check_r, int unit_r = 0,
                        const double* r_fixed = nullptr, double* Rhist = (double*)1, double* Shist = (double*)1,
                        int* status = nullptr) {
  cudaStream_t st = ctx->stream;
  if (Rhist == (double*)1) Rhist = ctx->Rhist.get();
  if (Shist == (double*)1) Shist = ctx->Shist.get();
  if (!status) status = ctx->status.get();
  if (ntile <= kScanSingleMax) {
    k_lag_scan<<<1, kScanThreads, 0, st>>>(ctx->tileA.get(), ctx->tileB.get(), ntile, ctx->OT.get(), ctx->scal.get(),
                                           Rhist, Shist, lag, check_r, status, unit_r, r_fixed, ctx->guide.get());
    LAUNCH_CHECK("k_lag_scan");
    COUNT_LAUNCH();
    return;
  }
  // long windows: the multi-CTA scan (k_scan_blocks / k_scan_mid / k_scan_ot / k_scan_guide)
  const int64_t nb = (ntile + kScanBlk - 1) / kScanBlk;
  ctx->scan_part.need(nb);
  ctx->scan_boff.need(nb);
  double* part = ctx->scan_part.get();
  if (!r_fixed && !unit_r)
    k_scan_blocks<<<(unsigned)nb, kScanThreads, 0, st>>>(ctx->tileA.get(), ctx->tileB.get(), ntile, ctx->scal.get(), 0,
                                                         part);
  k_scan_mid<<<1, kScanThreads, 0, st>>>(part, nb, 0, ctx->scal.get(), Rhist, Shist, lag, check_r, status, unit_r,
                                         r_fixed, ctx->scan_boff.get());
  k_scan_blocks<<<(unsigned)nb, kScanThreads, 0, st>>>(ctx->tileA.get(), ctx->tileB.get(), ntile, ctx->scal.get(), 1,
                                                       part);
  k_scan_mid<<<1, kScanThreads, 0, st>>>(part, nb, 1, ctx->scal.get(), Rhist, Shist, lag, check_r, status, unit_r,
                                         r_fixed, ctx->scan_boff.get());
  k_scan_ot<<<(unsigned)nb, kScanThreads, 0, st>>>(ctx->tileA.get(), ctx->tileB.get(), ntile, ctx->scal.get(),
                                                   ctx->scan_boff.get(), ctx->OT.get());
  k_scan_guide<<<(unsigned)((ntile + 255) / 256), 256, 0, st>>>(ctx->OT.get(), ntile, ctx->scal.get(), ctx->guide.get());
  LAUNCH_CHECK("k_scan");
  g_launches += 6;
}

static void launch_draw(tf_context* ctx, uint64_t seed, int64_t c, int64_t w, int64_t* idx,
                        double* wts, const uint64_t* seed_ptr = nullptr, PendState ps = PendState{}) {
  DrawArgs a{};
  a.ps = ps;
  a.shard = 0;
  a.accept = nullptr;
  a.seed_ptr = nullptr;
  a.seed = seed;
  a.seed_ptr = seed_ptr;
  a.c = c;
  a.scal = ctx->scal.get();
  a.OT = ctx->OT.get();
  a.guide = ctx->guide.get();
  a.ntile = (w + kPassTile - 1) / kPassTile;
  a.tA = ctx->tileA.get();
  a.tB = ctx->tileB.get();
  a.chunkA = ctx->chunkA.get();
  a.chunkB = ctx->chunkB.get();
  a.s = ctx->s.get();
  a.r = ctx->r.get();
  a.w = w;
  a.idx = idx;
  a.wts = wts;
  const int per = kDrawPerCta;
  k_draw<<<(unsigned)((c + per - 1) / per), kDrawThreads, 0, ctx->stream>>>(a);
  LAUNCH_CHECK("k_draw");
  COUNT_LAUNCH();
}

static void launch_fixed_weights(tf_context* ctx, const int64_t* idx, int64_t c, const double* s, const double* r,
                                 double* wts, PendState ps = PendState{}) {
  k_fixed_weights<<<(unsigned)((c + 255) / 256), 256, 0, ctx->stream>>>(idx, c, ctx->scal.get(), s, r, wts, ps);
  LAUNCH_CHECK("k_fixed_weights");
  COUNT_LAUNCH();
}

static void alloc_state(tf_context* ctx, int p_bar, int64_t c, int64_t w) {
  ctx->step_p = 0;  // the LsarDriver resident state is gone
  const int64_t ntile = (w + kPassTile - 1) / kPassTile;
  const int64_t nchunk = (w + kChunk - 1) / kChunk;
  ctx->s.need(w);
  ctx->r.need(w);
  ctx->chunkA.need(nchunk);
  ctx->chunkB.need(nchunk);
  ctx->tileA.need(ntile);
  ctx->tileB.need(ntile);
  ctx->OT.need(ntile);
  ctx->guide.need(guide_buckets(ntile) + 1);
  ctx->scal.need(4);
  ctx->Rhist.need(p_bar + 2);
  ctx->Shist.need(p_bar + 2);
  ctx->phi.need(p_bar + 1);
  ctx->coefs.need((size_t)p_bar * (p_bar + 1) / 2);
  ctx->taus.need(p_bar);
  ctx->idx.need(c);
  ctx->wts.need(c);
  ctx->status.need(4);
  ctx->method.need(p_bar);
  ctx->sb.flags.need(4);
  CK(cudaMemsetAsync(ctx->status.get(), 0, 4 * sizeof(int), ctx->stream));
  CK(cudaMemsetAsync(ctx->sb.flags.get(), 0, 4 * sizeof(int), ctx->stream));
}

static void ensure_events(tf_context* ctx, size_t n) {
  while (ctx->events.size() < n) {
    cudaEvent_t e;
    CK(cudaEventCreate(&e));
    ctx->events.push_back(e);
  }
}

static void ensure_span_events(tf_context* ctx) {
  if (!ctx->ev_begin) CK(cudaEventCreate(&ctx->ev_begin));
  if (!ctx->ev_end) CK(cudaEventCreate(&ctx->ev_end));
}

static void check_lsar_args(const tf_context* ctx, int p_bar, int64_t c) {
  // LsarDriver ctor (lsar.cpp:55-64)
  if (p_bar < 1) throw TfError{TF_USAGE, "maximum lag must be at least 1"};
  if (ctx->n == 0) throw TfError{TF_USAGE, "no series uploaded"};
  if (ctx->n <= (int64_t)p_bar + 1)
    throw TfError{TF_DATA, "series too short for maximum lag " + std::to_string(p_bar)};
  if (c < p_bar) throw TfError{TF_USAGE, "sample count below maximum lag"};
  // the fused pass stages a q-sample halo per tile in shared memory
  if (std::max(PassLayout(p_bar).bytes(), pass_smem_bytes(p_bar)) > (size_t)ctx->smem_optin_max)
    throw TfError{TF_USAGE, "maximum lag " + std::to_string(p_bar) + " exceeds the fused pass's shared-memory tile"};
}

// Run a fixed launch sequence through a CUDA graph: the first call for a
// shape runs eagerly, the second is captured (thread-local capture mode, so
// concurrent contexts on other host threads are unaffected), later calls
// replay the instantiated graph.  `capturing` tells the recorder to emit
// external event nodes for its timing events.  Returns the launch count.
template <class F>
static int64_t run_graphed(tf_context* ctx, GraphCache& gc, int64_t w, int64_t c, int p_bar, int mode,
                           bool& capturing, F&& record) {
  cudaStream_t st = ctx->stream;
  const bool same = gc.w == w && gc.c == c && gc.p_bar == p_bar && gc.mode == mode &&
                    gc.gen == g_alloc_gen.load();
  if (same && gc.exec) {
    CK(cudaGraphLaunch(gc.exec, st));
    g_launches += gc.launches;  // the replayed kernels count like launched ones
    return gc.launches;
  }
  if (same && gc.seen && !ctx->no_graphs) {
    const int64_t l0 = g_launches;
    cudaGraph_t graph = nullptr;
    CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    capturing = true;
    try {
      record();
    } catch (...) {
      capturing = false;
      cudaStreamEndCapture(st, &graph);
      if (graph) cudaGraphDestroy(graph);
      throw;
    }
    capturing = false;
    CK(cudaStreamEndCapture(st, &graph));
    // per-node priorities: the nodes captured from the low-priority side stream (k_fft_fold) must not
    // hold the SMs against the solve's kernels (by default every node takes the launch stream's priority)
    CK(cudaGraphInstantiateWithFlags(&gc.exec, graph, cudaGraphInstantiateFlagUseNodePriority));
    cudaGraphDestroy(graph);
    gc.launches = g_launches - l0;
    CK(cudaGraphLaunch(gc.exec, st));
    return gc.launches;
  }
  if (gc.exec) {
    cudaGraphExecDestroy(gc.exec);
    gc.exec = nullptr;
  }
  const int64_t l0 = g_launches;
  record();
  gc.w = w;
  gc.c = c;
  gc.p_bar = p_bar;
  gc.mode = mode;
  gc.seen = 1;
  gc.gen = g_alloc_gen.load();
  return g_launches - l0;
}

static void lsar_sweep(tf_context* ctx, int p_bar, int64_t c, uint64_t seed, const tf_lsar_diag* d,
                       double* taus, double* coefs, double* lag_seconds, int* p_star) {
  check_lsar_args(ctx, p_bar, c);
  const int64_t w = ctx->n - p_bar;  // constant row count (lsar.cpp:63)
  const int64_t ntile = (w + kPassTile - 1) / kPassTile;
  cudaStream_t st = ctx->stream;
  alloc_state(ctx, p_bar, c, w);
  // deterministic-index mode: reference indices, with the reference's weights
  // or (fixed_w null) the weights of this lag's own distribution
  const bool fixed = d && d->fixed_idx;
  const bool fixed_wts = fixed && d->fixed_w;
  if (fixed) {
    const size_t tot = (size_t)p_bar * c;
    for (size_t i = 0; i < tot; ++i)
      if (d->fixed_idx[i] < 0 || d->fixed_idx[i] >= w)
        throw TfError{TF_USAGE, "sample index out of range"};  // sketch.cpp:69
    ctx->fidx.need(tot);
    CK(cudaMemcpyAsync(ctx->fidx.get(), d->fixed_idx, tot * sizeof(int64_t), cudaMemcpyHostToDevice, st));
    if (fixed_wts) {
      ctx->fw.need(tot);
      CK(cudaMemcpyAsync(ctx->fw.get(), d->fixed_w, tot * sizeof(double), cudaMemcpyHostToDevice, st));
    }
  }
  const bool want_hist = d && (d->idx_out || d->w_out);
  if (want_hist) {
    ctx->idx_hist.need((size_t)p_bar * c);
    ctx->w_hist.need((size_t)p_bar * c);
  }
  reserve_exact(ctx, c, p_bar + 1);
  ctx->rank.need(p_bar);
  ctx->sweeps.need(p_bar);
  ensure_events(ctx, p_bar + 1);
  const bool phases = d && d->phase_seconds;
  while (phases && ctx->pev.size() < 2 * (size_t)p_bar) {
    cudaEvent_t e;
    CK(cudaEventCreate(&e));
    ctx->pev.push_back(e);
  }
  ensure_span_events(ctx);
  // per-lag draw seeds live in device memory, so a captured graph of the sweep
  // replays for any seed
  ctx->seedtab.need(p_bar + 1);
  {
    std::vector<uint64_t> seeds(p_bar + 1);
    for (int p = 0; p <= p_bar; ++p) seeds[p] = derive_seed(seed, (uint64_t)p);
    CK(cudaMemcpyAsync(ctx->seedtab.get(), seeds.data(), (p_bar + 1) * sizeof(uint64_t), cudaMemcpyHostToDevice, st));
    CK(cudaStreamSynchronize(st));  // the host vector goes out of scope
  }
  ctx->sb.M.need((size_t)c * ldq_of(2));  // the p = 1 Gram's dense staging (no allocation inside the loop)
  const bool use_fft = fft_sweep(ctx, p_bar);
  if (use_fft) reserve_fft(ctx, w);
  const FoldPlan fp = use_fft ? fold_plan(ctx, p_bar, w) : FoldPlan{};
  ctx->ymax.need(1);
  const unsigned long long* ybits = ctx->ymax.get();
  const int rn2 = d && d->rnorm2_out;
  bool capturing = false;
  // timing events: plain records when eager, external event nodes when captured
  auto rec = [&](cudaEvent_t e) {
    if (capturing) CK(cudaEventRecordWithFlags(e, st, cudaEventRecordExternal));
    else CK(cudaEventRecord(e, st));
  };
  auto record = [&]() {
    rec(ctx->ev_begin);
    rec(ctx->events[0]);
    // lag-0 pass: r_0 = -y[0..w), s_0 = 0  ->  s_1 = y^2 / sum y^2 (lsar.cpp:11-15)
    launch_pass(ctx, 0, w, ctx->phi.get(), ctx->scal.get());
    launch_absmax(ctx, w + p_bar, ybits);
    if (use_fft) launch_fft_series(ctx, w);  // series spectra for the FFT pass (once per sweep)
    for (int p = 1; p <= p_bar; ++p) {
      const int q = p - 1;
      launch_scan(ctx, ntile, q, 1);
      int64_t* idx = ctx->idx.get();
      double* wts = ctx->wts.get();
      if (fixed) {
        idx = ctx->fidx.get() + (size_t)(p - 1) * c;
        if (fixed_wts) wts = ctx->fw.get() + (size_t)(p - 1) * c;
        else launch_fixed_weights(ctx, idx, c, ctx->s.get(), ctx->r.get(), wts, pend_state(fp, p, ctx->Rhist.get()));
      } else {
        launch_draw(ctx, 0, c, w, idx, wts, ctx->seedtab.get() + p, pend_state(fp, p, ctx->Rhist.get()));
      }
      if (want_hist) {
        CK(cudaMemcpyAsync(ctx->idx_hist.get() + (size_t)(p - 1) * c, idx, c * sizeof(int64_t),
                           cudaMemcpyDeviceToDevice, st));
        CK(cudaMemcpyAsync(ctx->w_hist.get() + (size_t)(p - 1) * c, wts, c * sizeof(double),
                           cudaMemcpyDeviceToDevice, st));
      }
      if (phases) rec(ctx->pev[2 * (p - 1)]);
      // FFT lags with deferred folding: the score update of lag p needs nothing from the solve, so it
      // runs on the (low-priority) side stream beside it -- the solve's pivoted Cholesky and SVD leave
      // most SMs idle -- and the pass proper then only transforms and writes r_p
      // (a sweep that reports per-lag phase times keeps it on the main stream, inside the pass's
      // interval: those times are then the kernels' own, not what the overlap hides)
      const bool split = ctx->fft_split && fp.K > 1 && fft_lag(ctx, p_bar, p);
      const bool overlap = split && !phases;
      if (overlap) {
        CK(cudaEventRecord(ctx->ev_fork, st));
        CK(cudaStreamWaitEvent(ctx->side, ctx->ev_fork, 0));
        launch_fft_fold(ctx, p, w, ctx->scal.get(), fp, ctx->side);
        CK(cudaEventRecord(ctx->ev_join, ctx->side));
      }
      // rank-revealing solve of the sampled lag-p system (toeplitz.cpp:57-85)
      ExactOut o{ctx->phi.get(), ctx->coefs.get(), (int64_t)(p - 1) * p / 2, ctx->taus.get(), ctx->method.get(),
                 ctx->rank.get(), p, ctx->sweeps.get()};
      solve_exact(ctx, FwdRows{ctx->y.get(), idx, wts, 0}, c, p + 1, /*rev=*/0, o, nullptr, false, ybits);
      if (phases) rec(ctx->pev[2 * (p - 1) + 1]);
      if (overlap) CK(cudaStreamWaitEvent(st, ctx->ev_join, 0));
      else if (split) launch_fft_fold(ctx, p, w, ctx->scal.get(), fp, st);
      // residuals of the lag-p window fit + score update s_p = s_{p-1} + r_{p-1}^2/R_{p-1}
      if (fft_lag(ctx, p_bar, p)) launch_pass_fft(ctx, p, w, ctx->phi.get(), ctx->scal.get(), fp, split);
      else launch_pass(ctx, p, w, ctx->phi.get(), ctx->scal.get());
      rec(ctx->events[p]);
    }
    rec(ctx->ev_end);
    if (rn2) launch_scan(ctx, ntile, p_bar, 0);  // R_{p_bar} for the diagnostics
  };
  // The lag loop's launch sequence depends only on (w, c, p_bar, mode) and on
  // the buffers: graph capture/replay (run_graphed).
  const int mode = (fixed ? 1 : 0) | (want_hist ? 2 : 0) | (phases ? 4 : 0) | (rn2 ? 8 : 0) | (fixed_wts ? 16 : 0);
  const int64_t launches = run_graphed(ctx, ctx->lsar_graph, w, c, p_bar, mode, capturing, record);
  if (d && (d->scores_out || d->resid_out)) finish_fold(ctx, fp, p_bar, w);  // s_{p_bar}, r_{p_bar} into s / r
  CK(cudaStreamSynchronize(st));
  int sth[3];
  CK(cudaMemcpy(sth, ctx->status.get(), 3 * sizeof(int), cudaMemcpyDeviceToHost));
  raise_from_status(sth);
  std::vector<double> t(p_bar);
  CK(cudaMemcpy(t.data(), ctx->taus.get(), p_bar * sizeof(double), cudaMemcpyDeviceToHost));
  if (taus) std::memcpy(taus, t.data(), p_bar * sizeof(double));
  if (coefs)
    CK(cudaMemcpy(coefs, ctx->coefs.get(), sizeof(double) * (size_t)p_bar * (p_bar + 1) / 2,
                  cudaMemcpyDeviceToHost));
  if (lag_seconds)
    for (int p = 1; p <= p_bar; ++p) {
      float ms = 0.f;
      CK(cudaEventElapsedTime(&ms, ctx->events[p - 1], ctx->events[p]));
      lag_seconds[p - 1] = ms * 1e-3;
    }
  if (p_star) *p_star = tf_select_order(t.data(), p_bar, 1.96 / std::sqrt((double)c));
  if (d) {
    if (d->idx_out)
      CK(cudaMemcpy(d->idx_out, ctx->idx_hist.get(), sizeof(int64_t) * (size_t)p_bar * c, cudaMemcpyDeviceToHost));
    if (d->w_out)
      CK(cudaMemcpy(d->w_out, ctx->w_hist.get(), sizeof(double) * (size_t)p_bar * c, cudaMemcpyDeviceToHost));
    if (d->rnorm2_out)
      CK(cudaMemcpy(d->rnorm2_out, ctx->Rhist.get() + 1, sizeof(double) * p_bar, cudaMemcpyDeviceToHost));
    if (d->ssum_out)
      CK(cudaMemcpy(d->ssum_out, ctx->Shist.get() + 1, sizeof(double) * p_bar, cudaMemcpyDeviceToHost));
    if (d->scores_out) CK(cudaMemcpy(d->scores_out, ctx->s.get(), sizeof(double) * w, cudaMemcpyDeviceToHost));
    if (d->resid_out) CK(cudaMemcpy(d->resid_out, ctx->r.get(), sizeof(double) * w, cudaMemcpyDeviceToHost));
    if (d->method_out) CK(cudaMemcpy(d->method_out, ctx->method.get(), sizeof(int) * p_bar, cudaMemcpyDeviceToHost));
    if (d->rank_out) CK(cudaMemcpy(d->rank_out, ctx->rank.get(), sizeof(int) * p_bar, cudaMemcpyDeviceToHost));
    if (d->svd_sweeps_out)
      CK(cudaMemcpy(d->svd_sweeps_out, ctx->sweeps.get(), sizeof(int) * p_bar, cudaMemcpyDeviceToHost));
    if (d->launches_out) *d->launches_out = launches;
    if (phases)
      for (int p = 1; p <= p_bar; ++p) {
        float a = 0.f, b = 0.f, cc = 0.f;
        CK(cudaEventElapsedTime(&a, ctx->events[p - 1], ctx->pev[2 * (p - 1)]));
        CK(cudaEventElapsedTime(&b, ctx->pev[2 * (p - 1)], ctx->pev[2 * (p - 1) + 1]));
        CK(cudaEventElapsedTime(&cc, ctx->pev[2 * (p - 1) + 1], ctx->events[p]));
        d->phase_seconds[3 * (p - 1) + 0] = a * 1e-3;
        d->phase_seconds[3 * (p - 1) + 1] = b * 1e-3;
        d->phase_seconds[3 * (p - 1) + 2] = cc * 1e-3;
      }
  }
}

// ---------------------------------------------------------------------------
// Batched LSAR sweeps: B series of equal length n (or one series shared by B
// seeds: y_stride 0), the same p_bar and c -- the BASELINE C5 batch and the
// reference's multi-seed loops (run_compare / run_sweep, bench.cpp:183-188,
// 221-228).  Per lag four launches cover every series (blockIdx.y / x =
// series): the exact-tap-order pass (k_lsar_pass), the scan, the draws and
// the one-CTA solve k_bsolve (K <= 64).  Per-series state lives at fixed
// strides.  A series whose sampled system breaks down is flagged and re-run
// by the caller through the single-series path (lsar_sweep).
static constexpr int kBatchMaxPbar = kBsMaxK - 1;

static void lsar_batch(tf_context* ctx, const double* y_host, int64_t y_stride, int64_t B, int64_t n, int p_bar,
                       int64_t c, const uint64_t* seeds, const int64_t* fixed_idx, const double* fixed_w,
                       double* taus, double* coefs, double* lag_seconds, int* status_out, int* fallback_out) {
  if (B < 1) throw TfError{TF_USAGE, "batch must hold at least one series"};
  if (B > 65535) throw TfError{TF_USAGE, "batch exceeds 65535 fits per call (launch grid y limit)"};
  if (p_bar < 1) throw TfError{TF_USAGE, "maximum lag must be at least 1"};
  if (p_bar > kBatchMaxPbar)
    throw TfError{TF_USAGE, "batched sweeps support p_bar <= " + std::to_string(kBatchMaxPbar)};
  if (n <= (int64_t)p_bar + 1) throw TfError{TF_DATA, "series too short for maximum lag " + std::to_string(p_bar)};
  if (c < p_bar) throw TfError{TF_USAGE, "sample count below maximum lag"};
  if (y_stride != 0 && y_stride < n) throw TfError{TF_USAGE, "series stride below series length"};
  const int64_t w = n - p_bar;
  const int64_t ntile = (w + kPassTile - 1) / kPassTile;
  const int64_t nchunk = ntile * kChunksPerTile;
  const int64_t wst = ntile * kPassTile;                // state stride
  const int64_t nseries = y_stride ? B : 1;
  const int64_t yst = y_stride ? n + 64 : 0;            // device series stride (zero pad)
  const int G = guide_buckets(ntile);
  const int64_t ncoef = (int64_t)p_bar * (p_bar + 1) / 2;
  const bool fixed = fixed_idx && fixed_w;
  cudaStream_t st = ctx->stream;
  // ---- buffers ----
  ctx->bt_y.need((size_t)(nseries * (n + 64)));
  ctx->bt_s.need((size_t)(B * wst));
  ctx->bt_r.need((size_t)(B * wst));
  ctx->bt_cA.need((size_t)(B * nchunk));
  ctx->bt_cB.need((size_t)(B * nchunk));
  ctx->bt_tA.need((size_t)(B * ntile));
  ctx->bt_tB.need((size_t)(B * ntile));
  ctx->bt_OT.need((size_t)(B * ntile));
  ctx->bt_guide.need((size_t)(B * (G + 1)));
  ctx->bt_scal.need((size_t)(4 * B));
  ctx->bt_Rh.need((size_t)(B * (p_bar + 2)));
  ctx->bt_Sh.need((size_t)(B * (p_bar + 2)));
  ctx->bt_phi.need((size_t)(B * (p_bar + 1)));
  ctx->bt_coefs.need((size_t)(B * ncoef));
  ctx->bt_taus.need((size_t)(B * p_bar));
  ctx->bt_method.need((size_t)(B * p_bar));
  ctx->bt_S0.need((size_t)(B * kBsSLd * kBsSLd));
  ctx->bt_S1.need((size_t)(B * kBsSLd * kBsSLd));
  ctx->bt_status.need((size_t)(4 * B));
  ctx->bt_fb.need((size_t)B);
  ctx->bt_seed.need((size_t)((p_bar + 1) * B));
  if (fixed) {
    ctx->bt_fidx.need((size_t)(B * p_bar * c));
    ctx->bt_fw.need((size_t)(B * p_bar * c));
  } else {
    ctx->bt_idx.need((size_t)(B * c));
    ctx->bt_wts.need((size_t)(B * c));
  }
  // ---- inputs ----
  CK(cudaMemsetAsync(ctx->bt_y.get(), 0, (size_t)(nseries * (n + 64)) * sizeof(double), st));  // zero pads
  CK(cudaMemcpy2DAsync(ctx->bt_y.get(), (n + 64) * sizeof(double), y_host, (y_stride ? y_stride : n) * sizeof(double),
                       n * sizeof(double), (size_t)nseries, cudaMemcpyHostToDevice, st));
  CK(cudaMemsetAsync(ctx->bt_status.get(), 0, 4 * B * sizeof(int), st));
  CK(cudaMemsetAsync(ctx->bt_fb.get(), 0, B * sizeof(int), st));
  CK(cudaMemsetAsync(ctx->bt_scal.get(), 0, 4 * B * sizeof(double), st));
  std::vector<uint64_t> sd((size_t)(p_bar + 1) * B);  // [p][b] = derive_seed(seed_b, p)
  for (int p = 0; p <= p_bar; ++p)
    for (int64_t b = 0; b < B; ++b) sd[(size_t)p * B + b] = derive_seed(seeds[b], (uint64_t)p);
  CK(cudaMemcpyAsync(ctx->bt_seed.get(), sd.data(), sd.size() * sizeof(uint64_t), cudaMemcpyHostToDevice, st));
  if (fixed) {
    for (int64_t i = 0; i < B * p_bar * c; ++i)
      if (fixed_idx[i] < 0 || fixed_idx[i] >= w) throw TfError{TF_USAGE, "sample index out of range"};  // sketch.cpp:69
    CK(cudaMemcpyAsync(ctx->bt_fidx.get(), fixed_idx, B * p_bar * c * sizeof(int64_t), cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(ctx->bt_fw.get(), fixed_w, B * p_bar * c * sizeof(double), cudaMemcpyHostToDevice, st));
  }
  ensure_events(ctx, p_bar + 1);
  // ---- launches ----
  PassArgs pa{};
  pa.y = ctx->bt_y.get();
  pa.w = w;
  pa.s = ctx->bt_s.get();
  pa.r = ctx->bt_r.get();
  pa.chunkA = ctx->bt_cA.get();
  pa.chunkB = ctx->bt_cB.get();
  pa.tileA = ctx->bt_tA.get();
  pa.tileB = ctx->bt_tB.get();
  pa.ylen = n + 64;
  pa.bs_y = yst;
  pa.bs_w = wst;
  pa.bs_chunk = nchunk;
  pa.bs_tile = ntile;
  pa.bs_phi = p_bar + 1;
  pa.bs_scal = 4;
  pa.phi = ctx->bt_phi.get();
  pa.Rprev = ctx->bt_scal.get();
  const dim3 pgrid((unsigned)ntile, (unsigned)B);
  auto pass = [&](int q) {
    pa.q = q;
    const size_t smem = pass_smem_bytes(q);
    smem_optin((const void*)k_lsar_pass, smem);
    k_lsar_pass<<<pgrid, kPassThreads, smem, st>>>(pa);
    LAUNCH_CHECK("k_lsar_pass (batch)");
    COUNT_LAUNCH();
  };
  const size_t bsm = bsolve_smem_bytes();
  smem_optin((const void*)k_bsolve, bsm);
  CK(cudaEventRecord(ctx->events[0], st));
  pass(0);
  for (int p = 1; p <= p_bar; ++p) {
    const int q = p - 1;
    k_lag_scan<<<(unsigned)B, kScanThreads, 0, st>>>(ctx->bt_tA.get(), ctx->bt_tB.get(), ntile, ctx->bt_OT.get(),
                                                     ctx->bt_scal.get(), ctx->bt_Rh.get(), ctx->bt_Sh.get(), q, 1,
                                                     ctx->bt_status.get(), 0, nullptr, ctx->bt_guide.get(), ntile,
                                                     p_bar + 2);
    LAUNCH_CHECK("k_lag_scan (batch)");
    COUNT_LAUNCH();
    const int64_t* idx;
    const double* wts;
    int64_t bs_idx;
    if (fixed) {
      idx = ctx->bt_fidx.get() + (size_t)(p - 1) * c;
      wts = ctx->bt_fw.get() + (size_t)(p - 1) * c;
      bs_idx = (int64_t)p_bar * c;
    } else {
      DrawArgs da{};
      da.seed_ptr = ctx->bt_seed.get() + (size_t)p * B;
      da.bs_seed = 1;
      da.c = c;
      da.scal = ctx->bt_scal.get();
      da.OT = ctx->bt_OT.get();
      da.guide = ctx->bt_guide.get();
      da.ntile = ntile;
      da.tA = ctx->bt_tA.get();
      da.tB = ctx->bt_tB.get();
      da.chunkA = ctx->bt_cA.get();
      da.chunkB = ctx->bt_cB.get();
      da.s = ctx->bt_s.get();
      da.r = ctx->bt_r.get();
      da.w = w;
      da.idx = ctx->bt_idx.get();
      da.wts = ctx->bt_wts.get();
      da.bs_w = wst;
      da.bs_chunk = nchunk;
      da.bs_tile = ntile;
      const dim3 dgrid((unsigned)((c + kDrawPerCta - 1) / kDrawPerCta), (unsigned)B);
      k_draw<<<dgrid, kDrawThreads, 0, st>>>(da);
      LAUNCH_CHECK("k_draw (batch)");
      COUNT_LAUNCH();
      idx = ctx->bt_idx.get();
      wts = ctx->bt_wts.get();
      bs_idx = c;
    }
    BSolveArgs sa{};
    sa.y = ctx->bt_y.get();
    sa.bs_y = yst;
    sa.idx = idx;
    sa.wts = wts;
    sa.bs_idx = bs_idx;
    sa.c = c;
    sa.K = p + 1;
    sa.lag = p;
    sa.Sprev = (p & 1) ? ctx->bt_S0.get() : ctx->bt_S1.get();
    sa.Snext = (p & 1) ? ctx->bt_S1.get() : ctx->bt_S0.get();
    sa.phi = ctx->bt_phi.get();
    sa.bs_phi = p_bar + 1;
    sa.scal = ctx->bt_scal.get();
    sa.coefs = ctx->bt_coefs.get();
    sa.bs_coef = ncoef;
    sa.taus = ctx->bt_taus.get();
    sa.bs_tau = p_bar;
    sa.method = ctx->bt_method.get();
    sa.fallback = ctx->bt_fb.get();
    k_bsolve<<<(unsigned)B, kBsThreads, bsm, st>>>(sa);
    LAUNCH_CHECK("k_bsolve");
    COUNT_LAUNCH();
    pass(p);
    CK(cudaEventRecord(ctx->events[p], st));
  }
  CK(cudaStreamSynchronize(st));
  // ---- outputs ----
  std::vector<int> stv((size_t)(4 * B)), fb((size_t)B);
  CK(cudaMemcpy(stv.data(), ctx->bt_status.get(), stv.size() * sizeof(int), cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(fb.data(), ctx->bt_fb.get(), fb.size() * sizeof(int), cudaMemcpyDeviceToHost));
  if (taus) CK(cudaMemcpy(taus, ctx->bt_taus.get(), (size_t)(B * p_bar) * sizeof(double), cudaMemcpyDeviceToHost));
  if (coefs) CK(cudaMemcpy(coefs, ctx->bt_coefs.get(), (size_t)(B * ncoef) * sizeof(double), cudaMemcpyDeviceToHost));
  for (int64_t b = 0; b < B; ++b) {
    if (status_out)
      for (int k = 0; k < 3; ++k) status_out[3 * b + k] = stv[4 * b + k];
    if (fallback_out) fallback_out[b] = fb[b];
  }
  if (lag_seconds)
    for (int p = 1; p <= p_bar; ++p) {
      float ms = 0.f;
      CK(cudaEventElapsedTime(&ms, ctx->events[p - 1], ctx->events[p]));
      lag_seconds[p - 1] = ms * 1e-3;
    }
}

// ---------------------------------------------------------------------------
// single operations
__global__ void k_partials(const double* s, const double* r, int64_t w, double* chunkA,
                           double* chunkB, double* tileA, double* tileB) {
  // same reduction shape as k_lsar_pass for externally supplied (s, r)
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t i0 = (int64_t)blockIdx.x * kPassTile;
  const int rows = (int)min((int64_t)kPassTile, w - i0);
  double tA = 0.0, tB = 0.0;
  for (int u = 0; u < kPassR; ++u) {
    const int row = tid + kPassThreads * u;
    double sv = 0.0, rv = 0.0;
    if (row < rows) {
      sv = s[i0 + row];
      rv = r ? r[i0 + row] : 0.0;
    }
    const double cA = warp_sum(sv), cB = warp_sum(rv * rv);
    const int crow = kPassThreads * u + kChunk * warp;
    if (lane == 0 && crow < rows) {
      chunkA[(i0 + crow) / kChunk] = cA;
      chunkB[(i0 + crow) / kChunk] = cB;
    }
    tA += cA;
    tB += cB;
  }
  __shared__ double wA[4], wB[4];
  if (lane == 0) {
    wA[warp] = tA;
    wB[warp] = tB;
  }
  __syncthreads();
  if (tid == 0) {
    tileA[blockIdx.x] = ((wA[0] + wA[1]) + wA[2]) + wA[3];
    tileB[blockIdx.x] = ((wB[0] + wB[1]) + wB[2]) + wB[3];
  }
}

__global__ void k_set_unit(double* scal) {
  // scores without a residual term: R := 1 so that mass = s + 0 / 1 = s
  scal[0] = 1.0;
}

// apply_sample (sketch.cpp:61-79) through the same forward-order row loader
// the solve uses: lag column j of row t is column p - 1 - j, the target p.
__global__ void k_materialize(FwdRows ld, int64_t c, int p, int width, double* a, double* b) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.y + threadIdx.y;
  if (t >= c) return;
  for (int j = threadIdx.x; j <= width; j += blockDim.x) {
    if (j == width) b[t] = ld(t, p);
    else a[t * width + j] = ld(t, p - 1 - j);
  }
}

// first non-finite position (series.cpp:23-32 validation), on the device
__global__ void k_first_nonfinite(const double* __restrict__ y, int64_t n, unsigned long long* first) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    if (!isfinite(y[i])) atomicMin(first, (unsigned long long)i);
}

static void upload_series(tf_context* ctx, const double* y, int64_t n, bool device_src) {
  if (n < 1 || !y) throw TfError{TF_DATA, "series must contain at least one value"};
  ctx->n = 0;  // no valid series until the check below passes (also when the allocation fails)
  ctx->step_p = 0;
  ctx->y.need(n + 64);
  if (device_src)
    CK(cudaMemcpyAsync(ctx->y.get(), y, n * sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
  else
    CK(cudaMemcpyAsync(ctx->y.get(), y, n * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemsetAsync(ctx->y.get() + n, 0, 64 * sizeof(double), ctx->stream));
  if (!device_src) {  // the finiteness check runs at HBM speed after the copy (a host loop cost ~10 ms at n = 1e7)
    ctx->fincheck.need(1);
    CK(cudaMemsetAsync(ctx->fincheck.get(), 0xff, sizeof(unsigned long long), ctx->stream));
    const unsigned fgrid = (unsigned)std::min<int64_t>((n + 255) / 256, 8LL * ctx->sm_count);
    k_first_nonfinite<<<fgrid, 256, 0, ctx->stream>>>(ctx->y.get(), n, ctx->fincheck.get());
    LAUNCH_CHECK("k_first_nonfinite");
    unsigned long long first = 0;
    CK(cudaMemcpyAsync(&first, ctx->fincheck.get(), sizeof(first), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    if (first < (unsigned long long)n)
      throw TfError{TF_DATA, "series value at position " + std::to_string(first) + " is not finite"};
  }
  CK(cudaStreamSynchronize(ctx->stream));
  ctx->n = n;
}

// LsarDriver::first_lag / advance (lsar.hpp:65-84, lsar.cpp:70-98): one lag
// of the recursion on the resident series.  p == 1: scores from
// init_leverage_p1; p > 1: scores = leverage_update(s_in, r_in) of the given
// lag-(p-1) state (host vectors of w = n - p_bar values), or -- s_in == r_in ==
// NULL -- of the device-resident state the previous call left (stepping in
// order).  Then the draws of Rng(derive_seed(seed, p)), the rank-revealing
// solve, the lag-p residuals.  Outputs the lag-p state: the scores used at lag
// p, the residuals, phi (all nullable).
static void lsar_step(tf_context* ctx, int p_bar, int64_t c, uint64_t seed, int p, const double* s_in,
                      const double* r_in, double* s_out, double* r_out, double* phi_out, int* method_out) {
  check_lsar_args(ctx, p_bar, c);
  if (p < 1 || p > p_bar) throw TfError{TF_USAGE, "cannot advance past maximum lag"};  // lsar.cpp:90
  const int64_t w = ctx->n - p_bar;
  const int64_t ntile = (w + kPassTile - 1) / kPassTile;
  cudaStream_t st = ctx->stream;
  const bool resident = p > 1 && !s_in && !r_in;
  if (resident && !(ctx->step_p == p - 1 && ctx->step_w == w))
    throw TfError{TF_USAGE, "no resident lag-" + std::to_string(p - 1) + " state: pass the previous state"};
  if (p > 1 && !resident && (!s_in || !r_in)) throw TfError{TF_USAGE, "a lag-p state needs scores and residuals"};
  if (!resident) {
    alloc_state(ctx, p_bar, c, w);
  } else {
    CK(cudaMemsetAsync(ctx->status.get(), 0, 4 * sizeof(int), st));
  }
  ctx->step_p = 0;
  reserve_exact(ctx, c, p + 1);
  ctx->rank.need(p_bar);
  if (p == 1) {
    launch_pass(ctx, 0, w, ctx->phi.get(), ctx->scal.get());  // r_0 = -y, s_0 = 0 -> s_1 = y^2 / ||y||^2
  } else if (!resident) {
    CK(cudaMemcpyAsync(ctx->s.get(), s_in, w * sizeof(double), cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(ctx->r.get(), r_in, w * sizeof(double), cudaMemcpyHostToDevice, st));
    k_partials<<<(unsigned)ntile, kPassThreads, 0, st>>>(ctx->s.get(), ctx->r.get(), w, ctx->chunkA.get(),
                                                        ctx->chunkB.get(), ctx->tileA.get(), ctx->tileB.get());
    LAUNCH_CHECK("k_partials");
  }
  launch_scan(ctx, ntile, p - 1, 1);
  launch_draw(ctx, derive_seed(seed, (uint64_t)p), c, w, ctx->idx.get(), ctx->wts.get());
  ExactOut o{ctx->phi.get(), nullptr, 0, nullptr, ctx->method.get(), ctx->rank.get(), p, nullptr};
  solve_exact(ctx, FwdRows{ctx->y.get(), ctx->idx.get(), ctx->wts.get(), 0}, c, p + 1, /*rev=*/0, o);
  launch_pass(ctx, p, w, ctx->phi.get(), ctx->scal.get());  // s_p = s_{p-1} + r_{p-1}^2 / R_{p-1}, r_p
  CK(cudaStreamSynchronize(st));
  int sth[3];
  CK(cudaMemcpy(sth, ctx->status.get(), 3 * sizeof(int), cudaMemcpyDeviceToHost));
  raise_from_status(sth);
  if (s_out) CK(cudaMemcpy(s_out, ctx->s.get(), w * sizeof(double), cudaMemcpyDeviceToHost));
  if (r_out) CK(cudaMemcpy(r_out, ctx->r.get(), w * sizeof(double), cudaMemcpyDeviceToHost));
  if (phi_out) CK(cudaMemcpy(phi_out, ctx->phi.get(), p * sizeof(double), cudaMemcpyDeviceToHost));
  if (method_out) CK(cudaMemcpy(method_out, ctx->method.get() + (p - 1), sizeof(int), cudaMemcpyDeviceToHost));
  ctx->step_p = p;
  ctx->step_w = w;
}

static void residuals_op(tf_context* ctx, const double* y, int64_t n_used, int p, const double* phi,
                         double* r_out) {
  if (p < 1) throw TfError{TF_USAGE, "lag order must be at least 1"};
  if (n_used <= p) throw TfError{TF_DATA, "series window too short for lag order"};
  upload_series(ctx, y, n_used, false);
  const int64_t w = n_used - p;
  alloc_state(ctx, p, p, w);
  CK(cudaMemsetAsync(ctx->s.get(), 0, w * sizeof(double), ctx->stream));
  CK(cudaMemsetAsync(ctx->r.get(), 0, w * sizeof(double), ctx->stream));
  CK(cudaMemcpyAsync(ctx->phi.get(), phi, p * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
  k_set_unit<<<1, 1, 0, ctx->stream>>>(ctx->scal.get());
  launch_pass(ctx, p, w, ctx->phi.get(), ctx->scal.get(), /*exact_order=*/true);  // toeplitz.cpp:87-98 tap order
  CK(cudaMemcpyAsync(r_out, ctx->r.get(), w * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
}

static void sample_op(tf_context* ctx, const double* scores, int64_t n, int64_t c, uint64_t seed,
                      int64_t* idx_out, double* w_out) {
  if (n < 1) throw TfError{TF_DATA, "empty distribution"};
  if (c < 1) throw TfError{TF_USAGE, "sample count must be positive"};
  // sketch.cpp:25-32: entries non-negative, sequential sum within 1e-8 of 1
  double total = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    if (!(scores[i] >= 0.0)) throw TfError{TF_DATA, "distribution has a negative entry"};
    total += scores[i];
  }
  if (std::fabs(total - 1.0) > 1e-8) {
    char buf[96];
    std::snprintf(buf, sizeof buf, "distribution sums to %g, not 1", total);
    throw TfError{TF_DATA, buf};
  }
  const int64_t ntile = (n + kPassTile - 1) / kPassTile;
  alloc_state(ctx, 1, c, n);
  CK(cudaMemcpyAsync(ctx->s.get(), scores, n * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemsetAsync(ctx->r.get(), 0, n * sizeof(double), ctx->stream));
  k_partials<<<(unsigned)ntile, kPassThreads, 0, ctx->stream>>>(ctx->s.get(), ctx->r.get(), n,
                                                               ctx->chunkA.get(), ctx->chunkB.get(),
                                                               ctx->tileA.get(), ctx->tileB.get());
  LAUNCH_CHECK("k_partials");
  COUNT_LAUNCH();
  launch_scan(ctx, ntile, 0, 0, /*unit_r=*/1);  // no residual term: mass = s + 0 / 1
  launch_draw(ctx, seed, c, n, ctx->idx.get(), ctx->wts.get());
  CK(cudaMemcpyAsync(idx_out, ctx->idx.get(), c * sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaMemcpyAsync(w_out, ctx->wts.get(), c * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  int sth[3];
  CK(cudaMemcpy(sth, ctx->status.get(), 3 * sizeof(int), cudaMemcpyDeviceToHost));
  if (sth[0] != 0) {
    if (sth[2] == kReasonZeroScoreSum) throw TfError{TF_DATA, "distribution sums to 0, not 1"};
    raise_from_status(sth);
  }
}

static void check_sample(int64_t n_used, int p, const int64_t* idx, int64_t c) {
  if (p < 1) throw TfError{TF_USAGE, "lag order must be at least 1"};
  if (n_used <= p) throw TfError{TF_DATA, "series window too short for lag order"};
  if (c < 1) throw TfError{TF_USAGE, "empty system"};
  const int64_t rows = n_used - p;
  for (int64_t t = 0; t < c; ++t)
    if (idx[t] < 0 || idx[t] >= rows) throw TfError{TF_USAGE, "sample index out of range"};
}

static void apply_sample_op(tf_context* ctx, const double* y, int64_t n_used, int p,
                            const int64_t* idx, const double* w, int64_t c, int width, double* a_out,
                            double* b_out) {
  if (width < 1 || width > p) throw TfError{TF_USAGE, "invalid column width"};
  check_sample(n_used, p, idx, c);
  upload_series(ctx, y, n_used, false);
  ctx->idx.need(c);
  ctx->wts.need(c);
  DBuf<double> A, B;
  A.need((size_t)c * width);
  B.need(c);
  CK(cudaMemcpyAsync(ctx->idx.get(), idx, c * sizeof(int64_t), cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpyAsync(ctx->wts.get(), w, c * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
  FwdRows ld{ctx->y.get(), ctx->idx.get(), ctx->wts.get(), 0};
  dim3 blk(32, 8);
  k_materialize<<<(unsigned)((c + 7) / 8), blk, 0, ctx->stream>>>(ld, c, p, width, A.get(), B.get());
  LAUNCH_CHECK("k_materialize");
  COUNT_LAUNCH();
  CK(cudaMemcpyAsync(a_out, A.get(), sizeof(double) * c * width, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaMemcpyAsync(b_out, B.get(), sizeof(double) * c, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  A.release();
  B.release();
}

static void solve_sampled_op(tf_context* ctx, const double* y, int64_t n_used, int p,
                             const int64_t* idx, const double* w, int64_t c, double* phi_out,
                             int* method_out) {
  check_sample(n_used, p, idx, c);
  upload_series(ctx, y, n_used, false);
  alloc_state(ctx, p, c, 1);
  CK(cudaMemcpyAsync(ctx->idx.get(), idx, c * sizeof(int64_t), cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpyAsync(ctx->wts.get(), w, c * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
  reserve_exact(ctx, c, p + 1);
  ctx->rank.need(1);
  ExactOut o{ctx->phi.get(), nullptr, 0, nullptr, ctx->method.get(), ctx->rank.get(), 1, nullptr};
  solve_exact(ctx, FwdRows{ctx->y.get(), ctx->idx.get(), ctx->wts.get(), 0}, c, p + 1, /*rev=*/0, o);
  CK(cudaMemcpyAsync(phi_out, ctx->phi.get(), p * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  int m = 0;
  CK(cudaMemcpyAsync(&m, ctx->method.get(), sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  int sth[3];
  CK(cudaMemcpy(sth, ctx->status.get(), 3 * sizeof(int), cudaMemcpyDeviceToHost));
  raise_from_status(sth);
  if (method_out) *method_out = m;
}

// ---------------------------------------------------------------------------
// Repeated Halving (repeated_halving.cpp:126-232)

static unsigned grid_for(int64_t n, const tf_context* ctx) {
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, (int64_t)ctx->sm_count * 16));
}

// exclusive scan of int32 `in` (n) and f(i, excl, value) for every element
template <class F>
static void scan_apply(tf_context* ctx, const int* in, int64_t n, F f) {
  const int64_t nt = (n + kScanTileN - 1) / kScanTileN;
  ctx->rh_tsum.need(nt + 2);
  long long* ts = ctx->rh_tsum.get();
  k_scan_tile_sums<<<(unsigned)nt, kRhThreads, 0, ctx->stream>>>(in, n, ts);
  k_scan_top<<<1, 1024, 0, ctx->stream>>>(ts, nt, ts + nt + 1);
  k_scan_apply<F><<<(unsigned)nt, kRhThreads, 0, ctx->stream>>>(in, n, ts, f);
  LAUNCH_CHECK("scan_apply");
  g_launches += 3;
}

// one halving level: next = sorted first half of the partial shuffle of cur
// (cur == nullptr: the identity level 0)
static void rh_halve(tf_context* ctx, uint64_t seed, const int64_t* cur, int64_t size, int64_t* next) {
  const int64_t half = size / 2;
  cudaStream_t st = ctx->stream;
  int* J = ctx->rh_J.get();
  int* cnt = ctx->rh_cnt.get();
  int* fill = ctx->rh_fill.get();
  int* pick = ctx->rh_pick.get();
  int* rej = ctx->rh_flag.get();
  CK(cudaMemsetAsync(cnt, 0, size * sizeof(int), st));
  CK(cudaMemsetAsync(fill, 0, size * sizeof(int), st));
  CK(cudaMemsetAsync(pick, 0, size * sizeof(int), st));
  CK(cudaMemsetAsync(rej, 0, sizeof(int), st));
  k_halve_draw<<<grid_for(half, ctx), 256, 0, st>>>(seed, size, half, J, rej);
  k_halve_draw_serial<<<1, 32, 0, st>>>(seed, size, half, J, rej);
  k_halve_count<<<grid_for(half, ctx), 256, 0, st>>>(J, half, cnt);
  LAUNCH_CHECK("k_halve_draw");
  g_launches += 3;
  scan_apply(ctx, cnt, size, StartF{ctx->rh_start.get()});
  k_halve_scatter<<<grid_for(half, ctx), 256, 0, st>>>(J, half, ctx->rh_start.get(), fill, ctx->rh_bk.get());
  k_halve_bucket_sort<<<grid_for(size, ctx), 256, 0, st>>>(cnt, ctx->rh_start.get(), size, ctx->rh_bk.get());
  k_halve_resolve<<<grid_for(half, ctx), 256, 0, st>>>(J, half, cnt, ctx->rh_start.get(), ctx->rh_bk.get(), pick);
  LAUNCH_CHECK("k_halve_resolve");
  g_launches += 3;
  scan_apply(ctx, pick, size, CompactF{cur, next});
}

// S (TPU, K) = R^-1 of the CholeskyQR of the approximation rows (forward order)
static void rh_factor(tf_context* ctx, const FwdRows& ld, int64_t rows, int K, double* S) {
  SolveOut o{ctx->rh_phis.get(), nullptr, 0, nullptr, nullptr, 0, ctx->status.get()};
  solve_rows(ctx, ld, rows, K, o, nullptr, nullptr, S, 0, nullptr, nullptr, /*exact=*/true);
}

static void launch_draw_on(tf_context* ctx, const double* scores, int64_t w, uint64_t seed,
                           int64_t c, int64_t* idx, double* wts, const uint64_t* seed_ptr = nullptr) {
  DrawArgs a{};
  a.shard = 0;
  a.accept = nullptr;
  a.seed_ptr = seed_ptr;
  a.seed = seed;
  a.c = c;
  a.scal = ctx->scal.get();
  a.OT = ctx->OT.get();
  a.guide = ctx->guide.get();
  a.ntile = (w + kPassTile - 1) / kPassTile;
  a.tA = ctx->tileA.get();
  a.tB = ctx->tileB.get();
  a.chunkA = ctx->chunkA.get();
  a.chunkB = ctx->chunkB.get();
  a.s = scores;
  a.r = nullptr;
  a.w = w;
  a.idx = idx;
  a.wts = wts;
  const int per = kDrawPerCta;
  k_draw<<<(unsigned)((c + per - 1) / per), kDrawThreads, 0, ctx->stream>>>(a);
  LAUNCH_CHECK("k_draw");
  COUNT_LAUNCH();
}

// distribution state (chunk/tile partials, tile prefix, total) of plain scores
static void score_distribution(tf_context* ctx, const double* scores, int64_t w) {
  const int64_t ntile = (w + kPassTile - 1) / kPassTile;
  k_partials<<<(unsigned)ntile, kPassThreads, 0, ctx->stream>>>(scores, nullptr, w, ctx->chunkA.get(),
                                                               ctx->chunkB.get(), ctx->tileA.get(),
                                                               ctx->tileB.get());
  LAUNCH_CHECK("k_partials");
  COUNT_LAUNCH();
  launch_scan(ctx, ntile, 0, 0, /*unit_r=*/1);
}

template <class L, class WL, bool UPPER>
static void rowsq_attr() {
  smem_optin((const void*)k_rowsq<L, WL, UPPER>, kRowsqSmem);
}

// scores of every window row t in [0, rows): out[t] = ||x_t W||^2 (Hankel tiles)
// columns of W handled by DMMA tiles: a last tile of <= kTailMax columns goes
// to k_rowsq_tail instead (N = 129 sketch rows: 128 + 1)
static inline int rowsq_main_cols(int N) {
  const int rem = N % 64;
  return (N > 64 && rem != 0 && rem <= kTailMax) ? N - rem : N;
}

template <class L, class WL>
static void rowsq_tail(tf_context* ctx, const L& ld, int64_t rows, int K, const WL& wl, int N0, int N, double* out,
                       int add) {
  if (N0 >= N || rows <= 0) return;
  const int T = N - N0;
  const size_t smem = sizeof(double) * (size_t)K * T;
  auto go = [&](auto kern, int rw) {
    smem_optin((const void*)kern, smem);
    const int64_t wblocks = (rows + 32LL * rw - 1) / (32LL * rw);
    const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>((wblocks + 7) / 8, 8LL * ctx->sm_count));
    kern<<<grid, 256, smem, ctx->stream>>>(ld, rows, K, wl, N0, N, out, add);
  };
  if (T <= 2) go(k_rowsq_tail<L, WL, 2, 8>, 8);
  else if (T <= 12) go(k_rowsq_tail<L, WL, 12, 4>, 4);
  else go(k_rowsq_tail<L, WL, 16, 2>, 2);
  LAUNCH_CHECK("k_rowsq_tail");
  COUNT_LAUNCH();
}

template <class WL, bool UPPER>
static void rowsq_all_rows(tf_context* ctx, int64_t rows, int K, const WL& wl, int Nfull, double* out) {
  const int N = rowsq_main_cols(Nfull);
  const int ntiles = (N + 63) / 64;
  if (ntiles > 8) throw TfError{TF_USAGE, "row-score tiles > 8"};
  const size_t smem = rowsq_hankel_smem(K);
  smem_optin((const void*)k_rowsq_hankel<WL, UPPER>, smem);
  int per_sm = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_rowsq_hankel<WL, UPPER>, kHkThreads, smem));
  // one wave of CTAs split over the column tiles in proportion to each tile's
  // cost: (k-steps it runs) x (8-column fragments it holds + F), F = 16
  // (measured: a block's loads, barriers and epilogue cost about as much as
  // two full column tiles of DMMA) -- narrow last tiles and the triangular
  // final pass (tile j only needs k < 64 (j + 1)) get somewhat fewer CTAs
  const int total = std::max(ntiles, per_sm * ctx->sm_count);
  double wsum = 0.0, wj[9];
  for (int j = 0; j < ntiles; ++j) {
    const int kend = UPPER ? std::min(hk_kpad(K), hk_kpad(std::min(K, 64 * (j + 1)))) : hk_kpad(K);
    const int frags = std::min(8, (N - 64 * j + 7) / 8);
    wj[j] = (double)kend * (frags + 16.0);
    wsum += wj[j];
  }
  HkPlan plan;
  plan.ntiles = ntiles;
  plan.first[0] = 0;
  double acc = 0.0;
  for (int j = 0; j < ntiles; ++j) {
    acc += wj[j];
    const int want = (int)std::lround(acc / wsum * total);
    plan.first[j + 1] = std::max(plan.first[j] + 1, std::min(want, total - (ntiles - 1 - j)));
  }
  const int nparts = ntiles + (Nfull > N ? 1 : 0);
  ctx->rh_part.need((size_t)nparts * rows);
  k_rowsq_hankel<WL, UPPER><<<plan.first[ntiles], kHkThreads, smem, ctx->stream>>>(
      ctx->y.get(), ctx->n, rows, K, wl, N, plan, ctx->rh_part.get());
  LAUNCH_CHECK("k_rowsq_hankel");
  rowsq_tail(ctx, WinRows{ctx->y.get(), nullptr}, rows, K, wl, N, Nfull, ctx->rh_part.get() + (size_t)ntiles * rows, 0);
  k_rowsq_combine<<<grid_for(rows, ctx), 256, 0, ctx->stream>>>(ctx->rh_part.get(), rows, nparts, out);
  LAUNCH_CHECK("k_rowsq_combine");
  g_launches += 2;
}

static int64_t rh_default_base(int64_t c, int64_t k) {  // repeated_halving.hpp:67-70
  const int64_t logk = (int64_t)std::ceil(std::log((double)k + 1.0));
  return std::max<int64_t>(c, 10 * k * logk);
}

static void rh_sweep(tf_context* ctx, int p_bar, int64_t c, const tf_rh_cfg* cfg_in, uint64_t seed,
                     const tf_rh_diag* d, double* taus, double* coefs, double* lag_seconds,
                     double* upfront_seconds, int* p_star) {
  // rh_fit argument checks (repeated_halving.cpp:191-200)
  if (p_bar < 1) throw TfError{TF_USAGE, "maximum lag must be at least 1"};
  if (ctx->n == 0) throw TfError{TF_USAGE, "no series uploaded"};
  if (ctx->n <= (int64_t)p_bar + 1)
    throw TfError{TF_DATA, "series too short for maximum lag " + std::to_string(p_bar)};
  if (c < p_bar) throw TfError{TF_USAGE, "sample count below maximum lag"};
  const int64_t m = ctx->n - p_bar;
  const int K = p_bar + 1;
  tf_rh_cfg cfg;
  if (cfg_in) {
    cfg = *cfg_in;
  } else {  // RHConfig::defaults (repeated_halving.cpp:33-41)
    cfg.sample_count = c;
    cfg.base_threshold = rh_default_base(c, K);
    cfg.gaussian_rows = (int64_t)std::ceil(8.0 * std::log((double)std::max<int64_t>(m, 2)));
    cfg.seed = derive_seed(seed, 0x5c07e5ull);
  }
  // RHConfig::validate (repeated_halving.cpp:43-47)
  if (cfg.sample_count < 1) throw TfError{TF_USAGE, "sample count must be positive"};
  if (cfg.base_threshold < cfg.sample_count) throw TfError{TF_USAGE, "base threshold below sample count"};
  if (cfg.gaussian_rows < 1) throw TfError{TF_USAGE, "need at least one sketch row"};
  if (m >= (int64_t)INT32_MAX) throw TfError{TF_USAGE, "series too long for the halving index width"};
  const int64_t sc = cfg.sample_count;
  const int g = (int)cfg.gaussian_rows;
  // level sizes are deterministic: size_{l+1} = size_l / 2 while size_l > base
  std::vector<int64_t> lsz{m}, loff{0, 0};
  while (lsz.back() > cfg.base_threshold) {
    lsz.push_back(lsz.back() / 2);
    loff.push_back(loff.back() + lsz.back());
  }
  const int depth = (int)lsz.size() - 1;
  // levker_init row checks (repeated_halving.cpp:53-56)
  const int64_t base_rows = lsz[depth];
  if (base_rows < K || (depth > 0 && sc < K))
    throw TfError{TF_NUMERICAL, "reference matrix has too few rows"};
  const bool fixed = d && d->fixed_idx;
  const bool fixed_wts = fixed && d->fixed_w;
  const bool fixed_lv = d && d->fixed_levels;
  const bool fixed_up = d && d->fixed_up_idx && d->fixed_up_w;
  cudaStream_t st = ctx->stream;
  alloc_state(ctx, p_bar, c, m);
  // buffers
  const int64_t lvl_total = loff.back();
  ctx->rh_lvl.need(std::max<int64_t>(lvl_total, 1));
  if (depth > 0) {
    ctx->rh_J.need(m / 2 + 1);
    ctx->rh_bk.need(m / 2 + 1);
    ctx->rh_cnt.need(m);
    ctx->rh_start.need(m);
    ctx->rh_fill.need(m);
    ctx->rh_pick.need(m);
  }
  ctx->rh_flag.need(4);
  const int64_t arows_max = std::max(base_rows, sc);
  ctx->rh_aidx.need(std::max(arows_max, depth == 0 ? m : 0));
  ctx->rh_aw.need(std::max(arows_max, depth == 0 ? m : 0));
  ctx->rh_ones.need(std::max(arows_max, depth == 0 ? m : 0));
  ctx->rh_sidx.need(sc);
  ctx->rh_sw.need(sc);
  ctx->rh_scores.need(m);
  ctx->rh_S.need(tpu_size(K));
  ctx->rh_phis.need(K + 1);
  ctx->rh_rest.need(2);
  const int Kp = g + K;
  const int64_t max_norm = (int64_t)g * arows_max;
  if (depth > 0) {
    ctx->rh_norm.need(max_norm);
    ctx->rh_ok.need((max_norm / 2 + 1) * 135 / 100 + 4096);
    ctx->rh_Gp.need(tpu_size(Kp));
    ctx->rh_H0.need((size_t)g * K);
    ctx->rh_W.need((size_t)g * K);
    reserve_gram(ctx, arows_max, Kp);
  }
  reserve_solve(ctx, std::max(arows_max, std::max(c, depth == 0 ? m : 0)), K);
  ctx->rh_tsum.need((std::max(m, ((max_norm / 2 + 1) * 135 / 100 + 4096)) + kScanTileN - 1) / kScanTileN + 3);
  if (fixed) {
    const size_t tot = (size_t)p_bar * c;
    for (size_t i = 0; i < tot; ++i)
      if (d->fixed_idx[i] < 0 || d->fixed_idx[i] >= m) throw TfError{TF_USAGE, "sample index out of range"};
    ctx->fidx.need(tot);
    CK(cudaMemcpyAsync(ctx->fidx.get(), d->fixed_idx, tot * sizeof(int64_t), cudaMemcpyHostToDevice, st));
    if (fixed_wts) {
      ctx->fw.need(tot);
      CK(cudaMemcpyAsync(ctx->fw.get(), d->fixed_w, tot * sizeof(double), cudaMemcpyHostToDevice, st));
    }
  }
  if (fixed_lv && lvl_total > 0) {
    for (int64_t i = 0; i < lvl_total; ++i)
      if (d->fixed_levels[i] < 0 || d->fixed_levels[i] >= m) throw TfError{TF_USAGE, "level index out of range"};
    CK(cudaMemcpyAsync(ctx->rh_lvl.get(), d->fixed_levels, lvl_total * sizeof(int64_t), cudaMemcpyHostToDevice, st));
  }
  if (fixed_up && depth > 0) {
    const size_t tot = (size_t)depth * sc;
    ctx->rh_fup.need(tot);
    ctx->rh_fupw.need(tot);
    CK(cudaMemcpyAsync(ctx->rh_fup.get(), d->fixed_up_idx, tot * sizeof(int64_t), cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(ctx->rh_fupw.get(), d->fixed_up_w, tot * sizeof(double), cudaMemcpyHostToDevice, st));
  }
  const bool want_up = d && (d->up_idx_out || d->up_w_out) && depth > 0;
  if (want_up) {
    ctx->rh_fup.need((size_t)depth * sc);
    ctx->rh_fupw.need((size_t)depth * sc);
  }
  const bool want_hist = d && (d->idx_out || d->w_out);
  if (want_hist) {
    ctx->idx_hist.need((size_t)p_bar * c);
    ctx->w_hist.need((size_t)p_bar * c);
  }
  ensure_events(ctx, p_bar + 2);
  const int64_t launches0 = g_launches;
  ensure_span_events(ctx);
  CK(cudaEventRecord(ctx->ev_begin, st));
  CK(cudaEventRecord(ctx->events[0], st));
  const double* y = ctx->y.get();
  k_fill<<<grid_for(arows_max, ctx), 256, 0, st>>>(ctx->rh_ones.get(), std::max(arows_max, depth == 0 ? m : 0), 1.0);
  COUNT_LAUNCH();
  // ---- halving (repeated_halving.cpp:126-145) ----
  auto level_ptr = [&](int l) -> int64_t* { return l == 0 ? nullptr : ctx->rh_lvl.get() + loff[l]; };
  if (!fixed_lv)
    for (int l = 1; l <= depth; ++l)
      rh_halve(ctx, derive_seed(cfg.seed, 0x10000ull + (uint64_t)l), level_ptr(l - 1), lsz[l - 1], level_ptr(l));
  // ---- base approximation: unweighted rows of the last level ----
  int64_t arows = base_rows;
  const int64_t* aidx;
  if (depth == 0) {
    k_iota<<<grid_for(m, ctx), 256, 0, st>>>(ctx->rh_aidx.get(), m);
    COUNT_LAUNCH();
    aidx = ctx->rh_aidx.get();
  } else {
    aidx = level_ptr(depth);
  }
  const double* aw = ctx->rh_ones.get();
  // ---- upward pass (repeated_halving.cpp:146-180) ----
  for (int i = depth - 1; i >= 0; --i) {
    FwdRows B{y, aidx, aw, 0};
    rh_factor(ctx, B, arows, K, ctx->rh_S.get());
    // Gaussian sketch rows (g x arows), then GB = N^T B through the Gram of [N | B]
    const uint64_t gseed = derive_seed(cfg.seed, 0x20000ull + (uint64_t)i);
    const int64_t count = (int64_t)g * arows;
    const int64_t attempts = (count / 2 + 1) * 135 / 100 + 4096;
    k_polar_flags<<<grid_for(attempts, ctx), 256, 0, st>>>(gseed, attempts, ctx->rh_ok.get());
    COUNT_LAUNCH();
    scan_apply(ctx, ctx->rh_ok.get(), attempts, PolarF{gseed, count, ctx->rh_norm.get()});
    k_check_normals<<<1, 1, 0, st>>>(ctx->rh_tsum.get() + ((attempts + kScanTileN - 1) / kScanTileN) + 1,
                                     (count + 1) / 2, ctx->status.get());
    COUNT_LAUNCH();
    ConcatRows cr{ctx->rh_norm.get(), g, B};
    gram(ctx, cr, arows, Kp, ctx->rh_Gp.get(), nullptr);
    k_rh_h0<<<grid_for((int64_t)g * K, ctx), 256, 0, st>>>(ctx->rh_Gp.get(), Kp, g, ctx->rh_S.get(), K,
                                                          ctx->rh_H0.get());
    k_rh_w<<<grid_for((int64_t)g * K, ctx), 256, 0, st>>>(ctx->rh_H0.get(), ctx->rh_S.get(), K, g,
                                                         ctx->rh_W.get());
    g_launches += 2;
    // sketched scores of every row of level i
    const int64_t len = lsz[i];
    if (i == 0 && rowsq_hankel_smem(K) <= 200 * 1024) {
      rowsq_all_rows<DenseW, false>(ctx, len, K, DenseW{ctx->rh_W.get(), g}, g, ctx->rh_scores.get());
    } else {
      WinRows rows_i{y, level_ptr(i)};
      rowsq_attr<WinRows, DenseW, false>();
      const int gm = rowsq_main_cols(g);
      k_rowsq<WinRows, DenseW, false><<<(unsigned)((len + 63) / 64), kGramThreads, kRowsqSmem, st>>>(
          rows_i, len, K, DenseW{ctx->rh_W.get(), g}, gm, ctx->rh_scores.get());
      LAUNCH_CHECK("k_rowsq");
      COUNT_LAUNCH();
      rowsq_tail(ctx, rows_i, len, K, DenseW{ctx->rh_W.get(), g}, gm, g, ctx->rh_scores.get(), 1);
    }
    const int64_t* sidx = ctx->rh_sidx.get();
    const double* sw = ctx->rh_sw.get();
    if (fixed_up) {
      sidx = ctx->rh_fup.get() + (size_t)i * sc;
      sw = ctx->rh_fupw.get() + (size_t)i * sc;
    } else {
      score_distribution(ctx, ctx->rh_scores.get(), len);
      launch_draw_on(ctx, ctx->rh_scores.get(), len, derive_seed(cfg.seed, 0x30000ull + (uint64_t)i), sc,
                     ctx->rh_sidx.get(), ctx->rh_sw.get());
    }
    if (want_up && !fixed_up) {
      CK(cudaMemcpyAsync(ctx->rh_fup.get() + (size_t)i * sc, sidx, sc * sizeof(int64_t), cudaMemcpyDeviceToDevice, st));
      CK(cudaMemcpyAsync(ctx->rh_fupw.get() + (size_t)i * sc, sw, sc * sizeof(double), cudaMemcpyDeviceToDevice, st));
    }
    k_rh_compose<<<grid_for(sc, ctx), 256, 0, st>>>(sidx, sw, level_ptr(i), sc, ctx->rh_aidx.get(),
                                                   ctx->rh_aw.get());
    COUNT_LAUNCH();
    aidx = ctx->rh_aidx.get();
    aw = ctx->rh_aw.get();
    arows = sc;
  }
  // ---- final unsketched scores over all m rows (repeated_halving.cpp:182-189) ----
  {
    FwdRows B{y, aidx, aw, 0};
    rh_factor(ctx, B, arows, K, ctx->rh_S.get());
    if (rowsq_hankel_smem(K) <= 200 * 1024) {
      rowsq_all_rows<TpuW, true>(ctx, m, K, TpuW{ctx->rh_S.get(), K}, K, ctx->rh_scores.get());
    } else {
      rowsq_attr<WinRows, TpuW, true>();
      const int km = rowsq_main_cols(K);
      k_rowsq<WinRows, TpuW, true><<<(unsigned)((m + 63) / 64), kGramThreads, kRowsqSmem, st>>>(
          WinRows{y, nullptr}, m, K, TpuW{ctx->rh_S.get(), K}, km, ctx->rh_scores.get());
      LAUNCH_CHECK("k_rowsq");
      COUNT_LAUNCH();
      rowsq_tail(ctx, WinRows{y, nullptr}, m, K, TpuW{ctx->rh_S.get(), K}, km, K, ctx->rh_scores.get(), 1);
    }
    score_distribution(ctx, ctx->rh_scores.get(), m);
  }
  // ---- per-lag solves from the fixed distribution (repeated_halving.cpp:205-231) ----
  //      (a fixed launch sequence per shape: captured into a CUDA graph and
  //      replayed, per-lag seeds from a device table)
  ctx->seedtab.need(p_bar + 1);
  {
    std::vector<uint64_t> seeds(p_bar + 1);
    for (int p = 0; p <= p_bar; ++p) seeds[p] = derive_seed(seed, (uint64_t)p);
    CK(cudaMemcpyAsync(ctx->seedtab.get(), seeds.data(), (p_bar + 1) * sizeof(uint64_t), cudaMemcpyHostToDevice, st));
    CK(cudaStreamSynchronize(st));
  }
  reserve_exact(ctx, c, K);
  ctx->rank.need(p_bar);
  ctx->sweeps.need(p_bar);
  bool capturing = false;
  auto rec = [&](cudaEvent_t e) {
    if (capturing) CK(cudaEventRecordWithFlags(e, st, cudaEventRecordExternal));
    else CK(cudaEventRecord(e, st));
  };
  auto record_lags = [&]() {
    rec(ctx->events[1]);
    for (int p = 1; p <= p_bar; ++p) {
      int64_t* idx = ctx->idx.get();
      double* wts = ctx->wts.get();
      if (fixed) {
        idx = ctx->fidx.get() + (size_t)(p - 1) * c;
        if (fixed_wts) wts = ctx->fw.get() + (size_t)(p - 1) * c;
        else launch_fixed_weights(ctx, idx, c, ctx->rh_scores.get(), nullptr, wts);
      } else {
        launch_draw_on(ctx, ctx->rh_scores.get(), m, 0, c, idx, wts, ctx->seedtab.get() + p);
      }
      if (want_hist) {
        CK(cudaMemcpyAsync(ctx->idx_hist.get() + (size_t)(p - 1) * c, idx, c * sizeof(int64_t),
                           cudaMemcpyDeviceToDevice, st));
        CK(cudaMemcpyAsync(ctx->w_hist.get() + (size_t)(p - 1) * c, wts, c * sizeof(double),
                           cudaMemcpyDeviceToDevice, st));
      }
      // apply_sample(full, s, p) + solve_compressed (repeated_halving.cpp:221-222)
      ExactOut o{ctx->phi.get(), ctx->coefs.get(), (int64_t)(p - 1) * p / 2, ctx->taus.get(), ctx->method.get(),
                 ctx->rank.get(), p, ctx->sweeps.get()};
      solve_exact(ctx, RevRows{y, idx, wts, p_bar}, c, p + 1, /*rev=*/1, o);
      rec(ctx->events[p + 1]);
    }
    rec(ctx->ev_end);
  };
  const int lag_mode = (fixed ? 1 : 0) | (want_hist ? 2 : 0) | (fixed_wts ? 4 : 0);
  run_graphed(ctx, ctx->rh_graph, m, c, p_bar, lag_mode, capturing, record_lags);
  const int64_t launches = g_launches - launches0;
  CK(cudaStreamSynchronize(st));
  int sth[3];
  CK(cudaMemcpy(sth, ctx->status.get(), 3 * sizeof(int), cudaMemcpyDeviceToHost));
  if (sth[0] != 0 && sth[1] == 0 && sth[2] == kReasonCholFail)
    throw TfError{TF_NUMERICAL, "reference matrix is rank deficient"};
  raise_from_status(sth);
  std::vector<double> t(p_bar);
  CK(cudaMemcpy(t.data(), ctx->taus.get(), p_bar * sizeof(double), cudaMemcpyDeviceToHost));
  if (taus) std::memcpy(taus, t.data(), p_bar * sizeof(double));
  if (coefs)
    CK(cudaMemcpy(coefs, ctx->coefs.get(), sizeof(double) * (size_t)p_bar * (p_bar + 1) / 2,
                  cudaMemcpyDeviceToHost));
  if (upfront_seconds) {
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, ctx->events[0], ctx->events[1]));
    *upfront_seconds = ms * 1e-3;
  }
  if (lag_seconds)
    for (int p = 1; p <= p_bar; ++p) {
      float ms = 0.f;
      CK(cudaEventElapsedTime(&ms, ctx->events[p], ctx->events[p + 1]));
      lag_seconds[p - 1] = ms * 1e-3;
    }
  if (p_star) *p_star = tf_select_order(t.data(), p_bar, 1.96 / std::sqrt((double)c));
  if (d) {
    if (d->scores_out) CK(cudaMemcpy(d->scores_out, ctx->rh_scores.get(), sizeof(double) * m, cudaMemcpyDeviceToHost));
    if (d->depth_out) *d->depth_out = depth;
    if (d->launches_out) *d->launches_out = launches;
    if (d->method_out) CK(cudaMemcpy(d->method_out, ctx->method.get(), sizeof(int) * p_bar, cudaMemcpyDeviceToHost));
    if (d->rank_out) CK(cudaMemcpy(d->rank_out, ctx->rank.get(), sizeof(int) * p_bar, cudaMemcpyDeviceToHost));
    if (d->levels_out && lvl_total > 0)
      CK(cudaMemcpy(d->levels_out, ctx->rh_lvl.get(), sizeof(int64_t) * lvl_total, cudaMemcpyDeviceToHost));
    if (want_up && d->up_idx_out)
      CK(cudaMemcpy(d->up_idx_out, ctx->rh_fup.get(), sizeof(int64_t) * depth * sc, cudaMemcpyDeviceToHost));
    if (want_up && d->up_w_out)
      CK(cudaMemcpy(d->up_w_out, ctx->rh_fupw.get(), sizeof(double) * depth * sc, cudaMemcpyDeviceToHost));
    if (d->idx_out)
      CK(cudaMemcpy(d->idx_out, ctx->idx_hist.get(), sizeof(int64_t) * (size_t)p_bar * c, cudaMemcpyDeviceToHost));
    if (d->w_out)
      CK(cudaMemcpy(d->w_out, ctx->w_hist.get(), sizeof(double) * (size_t)p_bar * c, cudaMemcpyDeviceToHost));
  }
}

// ---------------------------------------------------------------------------
// Repeated Halving over a general row source (repeated_halving.hpp:17-23,
// 76-90; repeated_halving.cpp:54-180): rows reached through a host gather
// callback, staged into dense device buffers; the halving, the leverage
// kernel (rank check by the pivoted double-double Cholesky = CPQR rule,
// inverse factor by CholeskyQR), the Gaussian sketch and the row scores are
// the Toeplitz path's kernels over dense row loaders.

// CPQR rank of a dense reference matrix (rows x K) under Eigen's rule
// (threshold max(rows, K) eps); LeverageKernel's checks (repeated_halving.cpp:56-64)
static void leverage_rank_check(tf_context* ctx, const double* B, int64_t rows, int K) {
  if (rows < K) throw TfError{TF_NUMERICAL, "reference matrix has too few rows"};
  reserve_exact(ctx, rows, K + 1);
  ctx->rh_phis.need(K + 2);
  ctx->rank.need(1);
  ctx->method.need(1);
  ExactOut o{ctx->rh_phis.get(), nullptr, 0, nullptr, ctx->method.get(), ctx->rank.get(), 1, nullptr};
  solve_exact(ctx, DenseRowsZ{B, (int64_t)K, K}, rows, K + 1, /*rev=*/0, o);
  int rk = 0;
  CK(cudaMemcpyAsync(&rk, ctx->rank.get(), sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  if (rk != K) throw TfError{TF_NUMERICAL, "reference matrix is rank deficient"};
}

// scores of the `len` dense rows C (len x K) against the reference matrix B
// (brows x K): ||R^-T P^T x||^2 (g == 0) or ||G Q R^-T P^T x||^2 / g with the
// sketch's normals drawn from derive-seeded stream `gseed` (g x brows, column j
// of G = draws j g .. j g + g - 1, sketch.cpp:241-253)
static void dense_scores(tf_context* ctx, const double* C, int64_t len, const double* B, int64_t brows, int K, int g,
                         uint64_t gseed, double* out) {
  cudaStream_t st = ctx->stream;
  leverage_rank_check(ctx, B, brows, K);
  ctx->rh_S.need(tpu_size(K));
  ctx->rh_phis.need(K + 2);
  reserve_solve(ctx, brows, K);
  SolveOut so{ctx->rh_phis.get(), nullptr, 0, nullptr, nullptr, 0, ctx->status.get()};
  CK(cudaMemsetAsync(ctx->status.get(), 0, 4 * sizeof(int), st));
  DenseRows bl{B, (int64_t)K};
  solve_rows(ctx, bl, brows, K, so, nullptr, nullptr, ctx->rh_S.get(), 0, nullptr, nullptr, /*exact=*/true);
  DenseRows cl{C, (int64_t)K};
  if (g <= 0) {
    rowsq_attr<DenseRows, TpuW, true>();
    const int km = rowsq_main_cols(K);
    k_rowsq<DenseRows, TpuW, true><<<(unsigned)((len + 63) / 64), kGramThreads, kRowsqSmem, st>>>(
        cl, len, K, TpuW{ctx->rh_S.get(), K}, km, out);
    LAUNCH_CHECK("k_rowsq");
    rowsq_tail(ctx, cl, len, K, TpuW{ctx->rh_S.get(), K}, km, K, out, 1);
    return;
  }
  const int Kp = g + K;
  const int64_t count = (int64_t)g * brows;
  const int64_t attempts = (count / 2 + 1) * 135 / 100 + 4096;
  ctx->rh_norm.need(count);
  ctx->rh_ok.need(attempts);
  ctx->rh_tsum.need((attempts + kScanTileN - 1) / kScanTileN + 3);
  ctx->rh_Gp.need(tpu_size(Kp));
  ctx->rh_H0.need((size_t)g * K);
  ctx->rh_W.need((size_t)g * K);
  reserve_gram(ctx, brows, Kp);
  k_polar_flags<<<grid_for(attempts, ctx), 256, 0, st>>>(gseed, attempts, ctx->rh_ok.get());
  scan_apply(ctx, ctx->rh_ok.get(), attempts, PolarF{gseed, count, ctx->rh_norm.get()});
  k_check_normals<<<1, 1, 0, st>>>(ctx->rh_tsum.get() + ((attempts + kScanTileN - 1) / kScanTileN) + 1, (count + 1) / 2,
                                   ctx->status.get());
  ConcatRowsT<DenseRows> cr{ctx->rh_norm.get(), g, bl};
  gram(ctx, cr, brows, Kp, ctx->rh_Gp.get(), nullptr);
  k_rh_h0<<<grid_for((int64_t)g * K, ctx), 256, 0, st>>>(ctx->rh_Gp.get(), Kp, g, ctx->rh_S.get(), K, ctx->rh_H0.get());
  k_rh_w<<<grid_for((int64_t)g * K, ctx), 256, 0, st>>>(ctx->rh_H0.get(), ctx->rh_S.get(), K, g, ctx->rh_W.get());
  rowsq_attr<DenseRows, DenseW, false>();
  const int gm = rowsq_main_cols(g);
  k_rowsq<DenseRows, DenseW, false><<<(unsigned)((len + 63) / 64), kGramThreads, kRowsqSmem, st>>>(
      cl, len, K, DenseW{ctx->rh_W.get(), g}, gm, out);
  LAUNCH_CHECK("k_rowsq");
  rowsq_tail(ctx, cl, len, K, DenseW{ctx->rh_W.get(), g}, gm, g, out, 1);
  g_launches += 8;
}

static void generalized_leverage(tf_context* ctx, const double* c_rows, int64_t rows, int64_t c_cols, const double* b,
                                 int64_t brows, int64_t b_cols, int64_t g, uint64_t gseed, double* out) {
  if (c_cols != b_cols) throw TfError{TF_USAGE, "column count mismatch"};  // repeated_halving.cpp:100
  if (rows < 0 || brows < 0 || c_cols < 1) throw TfError{TF_USAGE, "empty matrix"};
  const int K = (int)c_cols;
  cudaStream_t st = ctx->stream;
  DBuf<double> C, B;
  C.need((size_t)std::max<int64_t>(rows, 1) * K);
  B.need((size_t)std::max<int64_t>(brows, 1) * K);
  CK(cudaMemcpyAsync(C.get(), c_rows, sizeof(double) * rows * K, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(B.get(), b, sizeof(double) * brows * K, cudaMemcpyHostToDevice, st));
  ctx->rh_scores.need(std::max<int64_t>(rows, 1));
  ctx->status.need(4);
  dense_scores(ctx, C.get(), rows, B.get(), brows, K, (int)g, gseed, ctx->rh_scores.get());
  CK(cudaMemcpyAsync(out, ctx->rh_scores.get(), sizeof(double) * rows, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  int sth[3];
  CK(cudaMemcpy(sth, ctx->status.get(), 3 * sizeof(int), cudaMemcpyDeviceToHost));
  raise_from_status(sth);
}

// repeated_halving(RowSource, RHConfig) (repeated_halving.cpp:126-180)
static void repeated_halving_src(tf_context* ctx, int64_t n, int64_t k, tf_gather_fn gather, void* user,
                                 const tf_rh_cfg* cfg, double* approx_out, int64_t cap, int64_t* arows_out,
                                 int* levels_out) {
  if (!cfg || !gather) throw TfError{TF_USAGE, "row source and config required"};
  if (cfg->sample_count < 1) throw TfError{TF_USAGE, "sample count must be positive"};
  if (cfg->base_threshold < cfg->sample_count) throw TfError{TF_USAGE, "base threshold below sample count"};
  if (cfg->gaussian_rows < 1) throw TfError{TF_USAGE, "need at least one sketch row"};
  if (n < 1) throw TfError{TF_USAGE, "empty source"};
  if (k < 1) throw TfError{TF_USAGE, "empty matrix"};
  if (n >= (int64_t)INT32_MAX) throw TfError{TF_USAGE, "source too long for the halving index width"};
  cudaStream_t st = ctx->stream;
  const int K = (int)k;
  const int64_t sc = cfg->sample_count;
  std::vector<int64_t> lsz{n}, loff{0, 0};
  while (lsz.back() > cfg->base_threshold) {
    lsz.push_back(lsz.back() / 2);
    loff.push_back(loff.back() + lsz.back());
  }
  const int depth = (int)lsz.size() - 1;
  const int64_t arows_final = depth > 0 ? sc : n;
  if (cap < arows_final) throw TfError{TF_USAGE, "approximation buffer too small"};
  ctx->rh_lvl.need(std::max<int64_t>(loff.back(), 1));
  if (depth > 0) {
    ctx->rh_J.need(n / 2 + 1);
    ctx->rh_bk.need(n / 2 + 1);
    ctx->rh_cnt.need(n);
    ctx->rh_start.need(n);
    ctx->rh_fill.need(n);
    ctx->rh_pick.need(n);
    ctx->rh_tsum.need((n + kScanTileN - 1) / kScanTileN + 3);
  }
  ctx->rh_flag.need(4);
  ctx->status.need(4);
  CK(cudaMemsetAsync(ctx->status.get(), 0, 4 * sizeof(int), st));
  auto level_ptr = [&](int l) -> int64_t* { return l == 0 ? nullptr : ctx->rh_lvl.get() + loff[l]; };
  for (int l = 1; l <= depth; ++l)
    rh_halve(ctx, derive_seed(cfg->seed, 0x10000ull + (uint64_t)l), level_ptr(l - 1), lsz[l - 1], level_ptr(l));
  std::vector<int64_t> lv((size_t)std::max<int64_t>(loff.back(), 1));
  if (depth > 0)
    CK(cudaMemcpyAsync(lv.data(), ctx->rh_lvl.get(), sizeof(int64_t) * loff.back(), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  auto level_rows = [&](int l, std::vector<int64_t>& out) {  // global row ids of level l
    out.resize((size_t)lsz[l]);
    if (l == 0) std::iota(out.begin(), out.end(), int64_t(0));
    else std::copy(lv.begin() + loff[l], lv.begin() + loff[l] + lsz[l], out.begin());
  };
  // base approximation: the last level's rows (unweighted)
  std::vector<int64_t> ids;
  level_rows(depth, ids);
  std::vector<double> host((size_t)ids.size() * K);
  gather(user, ids.data(), (int64_t)ids.size(), host.data());
  DBuf<double> approx, rowsbuf;
  approx.need((size_t)std::max<int64_t>(std::max<int64_t>(lsz[depth], sc), 1) * K);
  CK(cudaMemcpyAsync(approx.get(), host.data(), sizeof(double) * host.size(), cudaMemcpyHostToDevice, st));
  int64_t arows = lsz[depth];
  std::vector<int64_t> sidx((size_t)sc);
  std::vector<double> sw((size_t)sc);
  for (int i = depth - 1; i >= 0; --i) {
    // scores of level i's rows against the approximation (8192-row blocks in
    // the reference; one block here), sketched with g mixes
    level_rows(i, ids);
    const int64_t len = (int64_t)ids.size();
    host.resize((size_t)len * K);
    gather(user, ids.data(), len, host.data());
    rowsbuf.need((size_t)len * K);
    CK(cudaMemcpyAsync(rowsbuf.get(), host.data(), sizeof(double) * host.size(), cudaMemcpyHostToDevice, st));
    ctx->rh_scores.need(len);
    dense_scores(ctx, rowsbuf.get(), len, approx.get(), arows, K, (int)cfg->gaussian_rows,
                 derive_seed(cfg->seed, 0x20000ull + (uint64_t)i), ctx->rh_scores.get());
    // leverage_to_distribution + sample_rows (sketch.cpp:20-59)
    alloc_state(ctx, 1, sc, len);
    score_distribution(ctx, ctx->rh_scores.get(), len);
    launch_draw_on(ctx, ctx->rh_scores.get(), len, derive_seed(cfg->seed, 0x30000ull + (uint64_t)i), sc,
                   ctx->idx.get(), ctx->wts.get());
    CK(cudaMemcpyAsync(sidx.data(), ctx->idx.get(), sizeof(int64_t) * sc, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(sw.data(), ctx->wts.get(), sizeof(double) * sc, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    int sth[3];
    CK(cudaMemcpy(sth, ctx->status.get(), 3 * sizeof(int), cudaMemcpyDeviceToHost));
    raise_from_status(sth);
    // picked rows, weighted: the next approximation
    std::vector<int64_t> picked((size_t)sc);
    for (int64_t t = 0; t < sc; ++t) picked[t] = ids[(size_t)sidx[t]];
    host.resize((size_t)sc * K);
    gather(user, picked.data(), sc, host.data());
    for (int64_t t = 0; t < sc; ++t)
      for (int j = 0; j < K; ++j) host[(size_t)t * K + j] *= sw[t];
    CK(cudaMemcpyAsync(approx.get(), host.data(), sizeof(double) * host.size(), cudaMemcpyHostToDevice, st));
    arows = sc;
  }
  CK(cudaMemcpyAsync(approx_out, approx.get(), sizeof(double) * arows * K, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (arows_out) *arows_out = arows;
  if (levels_out) *levels_out = depth;
}

// ---------------------------------------------------------------------------
// Row-sharded LSAR steps.  The caller (paper_2112_12994_b200/
// shard.py) owns the collectives: per lag an allgather of this shard's
// (sum s, sum r^2) and, per CholeskyQR pass, an allreduce of the K x K Gram.
// The shard's series slice is y[row0 .. row0 + w_local + p_bar) (uploaded with
// tf_upload_series); its window rows are the global rows row0 .. row0 + w_local.

__global__ void k_sum_tiles(const double* tA, const double* tB, int64_t ntile, double* out) {
  __shared__ double ra[1024], rb[1024];
  const int tid = threadIdx.x;
  const int64_t seg = (ntile + 1023) / 1024;
  const int64_t b = min(ntile, (int64_t)tid * seg), e = min(ntile, b + seg);
  double sa = 0.0, sb = 0.0;
  for (int64_t t = b; t < e; ++t) {
    sa += tA[t];
    sb += tB[t];
  }
  ra[tid] = sa;
  rb[tid] = sb;
  __syncthreads();
  for (int o = 512; o > 0; o >>= 1) {
    if (tid < o) {
      ra[tid] = ra[tid] + ra[tid + o];
      rb[tid] = rb[tid] + rb[tid + o];
    }
    __syncthreads();
  }
  if (tid == 0) {
    out[0] = ra[0];
    out[1] = rb[0];
  }
}

struct CompactDrawF {
  const int64_t* idx;
  const double* wts;
  int64_t* oidx;
  double* ow;
  __device__ void operator()(int64_t t, long long excl, int v) const {
    if (v) {
      oidx[excl] = idx[t];
      ow[excl] = wts[t];
    }
  }
};

static void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) throw TfError{TF_NCCL, std::string(what) + ": " + ncclGetErrorString(r)};
}

static void nccl_init(tf_context* ctx, const unsigned char* id, int world, int rank) {
  if (world < 1 || rank < 0 || rank >= world) throw TfError{TF_USAGE, "invalid rank / world size"};
  if (ctx->comm) {
    ncclCommDestroy(ctx->comm);
    ctx->comm = nullptr;
  }
  ncclUniqueId uid;
  std::memcpy(&uid, id, sizeof uid);
  nccl_check(ncclCommInitRank(&ctx->comm, world, uid, rank), "ncclCommInitRank");
  ctx->nc_world = world;
  ctx->nc_rank = rank;
}

// keep y[start, start + len) of the resident series (a shard's slice + halo)
static void keep_slice(tf_context* ctx, int64_t start, int64_t len) {
  if (start < 0 || len < 1 || start + len > ctx->n) throw TfError{TF_USAGE, "slice outside the resident series"};
  tfe::DBuf<double> tmp;
  tmp.need(len + 64);
  CK(cudaMemcpyAsync(tmp.get(), ctx->y.get() + start, len * sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
  CK(cudaMemsetAsync(tmp.get() + len, 0, 64 * sizeof(double), ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  std::swap(ctx->y.p, tmp.p);
  std::swap(ctx->y.n, tmp.n);
  ctx->n = len;
  g_alloc_gen.fetch_add(1);
}

// Row-sharded LSAR sweep of one long series, one process per
// GPU: this context holds window rows [row0, row0 + w) of the global window as
// the slice y[row0 .. row0 + w + p_bar) (uploaded / kept with tf_keep_slice).
// Per lag, on the context stream, with no host synchronisation (the lag loop
// is graph-captured, NCCL included):
//   local fused pass -> (sum s, sum r^2) -> ncclAllGather -> k_shard_scal
//   (global R, this shard's CDF segment) -> local scan with the global R ->
//   the draws of Rng(derive_seed(seed, p)) that land in the segment, compacted
//   in draw order -> double-double Gram of the local sampled rows ->
//   ncclAllGather of the partials -> rank-ordered double-double sum -> the
//   rank-revealing solve, identical on every rank -> phi for the next pass.
static void lsar_sweep_sharded(tf_context* ctx, int p_bar, int64_t c, uint64_t seed, const tf_lsar_diag* d,
                               double* taus, double* coefs, double* lag_seconds, int* p_star) {
  if (!ctx->comm) throw TfError{TF_USAGE, "no NCCL communicator (tf_nccl_init)"};
  if (p_bar < 1) throw TfError{TF_USAGE, "maximum lag must be at least 1"};
  if (ctx->n == 0) throw TfError{TF_USAGE, "no series uploaded"};
  if (ctx->n <= (int64_t)p_bar) throw TfError{TF_DATA, "shard slice shorter than its rows plus the p_bar halo"};
  if (c < p_bar) throw TfError{TF_USAGE, "sample count below maximum lag"};
  if (d && d->fixed_idx) throw TfError{TF_USAGE, "deterministic-index mode is single-shard only"};
  const int world = ctx->nc_world, rank = ctx->nc_rank;
  const int64_t w = ctx->n - p_bar;  // this shard's window rows
  const int64_t ntile = (w + kPassTile - 1) / kPassTile;
  const int K = p_bar + 1;
  cudaStream_t st = ctx->stream;
  alloc_state(ctx, p_bar, c, w);
  reserve_exact(ctx, c, K);
  ctx->rank.need(p_bar);
  ctx->sweeps.need(p_bar);
  ctx->sh_part.need(2);
  ctx->sh_gath.need((size_t)3 * world);
  ctx->sh_par.need(4);
  ctx->sh_dummy.need(4);
  ctx->sh_idx.need(c);
  ctx->sh_wts.need(c);
  ctx->rh_ok.need(c);
  ctx->rh_tsum.need((c + kScanTileN - 1) / kScanTileN + 3);
  ctx->sb.Gloc.need((size_t)2 * K * K);
  ctx->sb.Gg.need((size_t)2 * K * K * world);
  ensure_events(ctx, p_bar + 1);
  ensure_span_events(ctx);
  const bool phases = d && d->phase_seconds;
  while (phases && ctx->pev.size() < 2 * (size_t)p_bar) {
    cudaEvent_t e;
    CK(cudaEventCreate(&e));
    ctx->pev.push_back(e);
  }
  ctx->seedtab.need(p_bar + 1);
  {
    std::vector<uint64_t> seeds(p_bar + 1);
    for (int p = 0; p <= p_bar; ++p) seeds[p] = derive_seed(seed, (uint64_t)p);
    CK(cudaMemcpyAsync(ctx->seedtab.get(), seeds.data(), (p_bar + 1) * sizeof(uint64_t), cudaMemcpyHostToDevice, st));
    CK(cudaStreamSynchronize(st));
  }
  CK(cudaMemsetAsync(ctx->sh_par.get(), 0, 4 * sizeof(double), st));
  const bool use_fft = fft_sweep(ctx, p_bar);
  if (use_fft) reserve_fft(ctx, w);
  const FoldPlan fp = use_fft ? fold_plan(ctx, p_bar, w) : FoldPlan{};
  ctx->ymax.need(1);
  const unsigned long long* ybits = ctx->ymax.get();
  const int64_t nt = (c + kScanTileN - 1) / kScanTileN;
  const long long* kdev = ctx->rh_tsum.get() + nt + 1;  // this shard's draw count (scan_apply total)
  bool capturing = false;
  auto rec = [&](cudaEvent_t e) {
    if (capturing) CK(cudaEventRecordWithFlags(e, st, cudaEventRecordExternal));
    else CK(cudaEventRecord(e, st));
  };
  // The score update beside the solve (k_fft_fold on the side stream) in the sharded loop: measured at
  // C4 through one rank, the captured graph loses the overlap (5.22 s; 4.93 s with the update fused into
  // the pass) while eager launches keep it (4.62 s) -- the graph's NCCL nodes seem to serialise the
  // side branch.  So shards long enough that a lag's device time dwarfs its ~25 launches run the lag
  // loop eagerly with the overlap; shorter ones replay the graph with the fused update.
  const bool sh_split = ctx->fft_split && use_fft && fp.K > 1 && w >= ((int64_t)1 << 24);
  auto record = [&]() {
    rec(ctx->ev_begin);
    rec(ctx->events[0]);
    launch_pass(ctx, 0, w, ctx->phi.get(), ctx->sh_par.get());  // r_0 = -y, s_0 = 0
    launch_absmax(ctx, w + p_bar, ybits);
    if (use_fft) launch_fft_series(ctx, w);
    for (int p = 1; p <= p_bar; ++p) {
      const int q = p - 1;
      k_sum_tiles<<<1, 1024, 0, st>>>(ctx->tileA.get(), ctx->tileB.get(), ntile, ctx->sh_part.get());
      nccl_check(ncclAllGather(ctx->sh_part.get(), ctx->sh_gath.get(), 2, ncclDouble, ctx->comm, st), "ncclAllGather");
      k_shard_R<<<1, 1, 0, st>>>(ctx->sh_gath.get(), world, ctx->sh_par.get(), ctx->Rhist.get(), q,
                                 ctx->status.get());
      // local CDF with the global R (its total S_local lands in scal[1])
      launch_scan(ctx, ntile, q, 0, 0, ctx->sh_par.get(), nullptr, nullptr, ctx->sh_dummy.get());
      nccl_check(ncclAllGather(ctx->scal.get() + 1, ctx->sh_gath.get() + 2 * world, 1, ncclDouble, ctx->comm, st),
                 "ncclAllGather");
      k_shard_seg<<<1, 1, 0, st>>>(ctx->sh_gath.get() + 2 * world, world, rank, ctx->sh_par.get(), ctx->Shist.get(), q,
                                   ctx->status.get());
      g_launches += 3;
      DrawArgs a{};
      a.seed_ptr = ctx->seedtab.get() + p;
      a.c = c;
      a.scal = ctx->scal.get();
      a.OT = ctx->OT.get();
      a.guide = ctx->guide.get();
      a.ntile = ntile;
      a.tA = ctx->tileA.get();
      a.tB = ctx->tileB.get();
      a.chunkA = ctx->chunkA.get();
      a.chunkB = ctx->chunkB.get();
      a.s = ctx->s.get();
      a.r = ctx->r.get();
      a.w = w;
      a.idx = ctx->idx.get();
      a.wts = ctx->wts.get();
      a.shard = 1;
      a.par = ctx->sh_par.get();
      a.accept = ctx->rh_ok.get();
      a.ps = pend_state(fp, p, ctx->Rhist.get());
      k_draw<<<(unsigned)((c + kDrawPerCta - 1) / kDrawPerCta), kDrawThreads, 0, st>>>(a);
      LAUNCH_CHECK("k_draw (shard)");
      COUNT_LAUNCH();
      // this shard's draws in draw order (deterministic local row order)
      scan_apply(ctx, ctx->rh_ok.get(), c, CompactDrawF{ctx->idx.get(), ctx->wts.get(), ctx->sh_idx.get(),
                                                        ctx->sh_wts.get()});
      if (phases) rec(ctx->pev[2 * (p - 1)]);
      // the shard's score update of an FFT lag beside the (replicated) solve, as in lsar_sweep
      const bool split = sh_split && fft_lag(ctx, p_bar, p);
      const bool overlap = split && !phases;
      if (overlap) {
        CK(cudaEventRecord(ctx->ev_fork, st));
        CK(cudaStreamWaitEvent(ctx->side, ctx->ev_fork, 0));
        launch_fft_fold(ctx, p, w, ctx->sh_par.get(), fp, ctx->side);
        CK(cudaEventRecord(ctx->ev_join, ctx->side));
      }
      ExactOut o{ctx->phi.get(), ctx->coefs.get(), (int64_t)(p - 1) * p / 2, ctx->taus.get(), ctx->method.get(),
                 ctx->rank.get(), p, ctx->sweeps.get()};
      solve_exact(ctx, FwdRows{ctx->y.get(), ctx->sh_idx.get(), ctx->sh_wts.get(), 0}, c, p + 1, /*rev=*/0, o, kdev,
                  /*sharded=*/true, ybits);
      if (phases) rec(ctx->pev[2 * (p - 1) + 1]);
      if (overlap) CK(cudaStreamWaitEvent(st, ctx->ev_join, 0));
      else if (split) launch_fft_fold(ctx, p, w, ctx->sh_par.get(), fp, st);
      if (fft_lag(ctx, p_bar, p)) launch_pass_fft(ctx, p, w, ctx->phi.get(), ctx->sh_par.get(), fp, split);
      else launch_pass(ctx, p, w, ctx->phi.get(), ctx->sh_par.get());  // R_{p-1} = par[0]
      rec(ctx->events[p]);
    }
    rec(ctx->ev_end);
  };
  const int mode = 64 | (phases ? 4 : 0);
  const bool graphs_off = ctx->no_graphs;
  ctx->no_graphs = graphs_off || sh_split;  // the overlapped sweep is launched eagerly (see sh_split)
  int64_t launches = 0;
  try {
    launches = run_graphed(ctx, ctx->lsar_graph, w, c, p_bar, mode, capturing, record);
  } catch (...) {
    ctx->no_graphs = graphs_off;
    throw;
  }
  ctx->no_graphs = graphs_off;
  CK(cudaStreamSynchronize(st));
  int sth[3];
  CK(cudaMemcpy(sth, ctx->status.get(), 3 * sizeof(int), cudaMemcpyDeviceToHost));
  raise_from_status(sth);
  std::vector<double> t(p_bar);
  CK(cudaMemcpy(t.data(), ctx->taus.get(), p_bar * sizeof(double), cudaMemcpyDeviceToHost));
  if (taus) std::memcpy(taus, t.data(), p_bar * sizeof(double));
  if (coefs)
    CK(cudaMemcpy(coefs, ctx->coefs.get(), sizeof(double) * (size_t)p_bar * (p_bar + 1) / 2, cudaMemcpyDeviceToHost));
  if (lag_seconds)
    for (int p = 1; p <= p_bar; ++p) {
      float ms = 0.f;
      CK(cudaEventElapsedTime(&ms, ctx->events[p - 1], ctx->events[p]));
      lag_seconds[p - 1] = ms * 1e-3;
    }
  if (p_star) *p_star = tf_select_order(t.data(), p_bar, 1.96 / std::sqrt((double)c));
  if (d) {
    if (d->rnorm2_out) CK(cudaMemcpy(d->rnorm2_out, ctx->Rhist.get() + 1, sizeof(double) * p_bar, cudaMemcpyDeviceToHost));
    if (d->ssum_out) CK(cudaMemcpy(d->ssum_out, ctx->Shist.get() + 1, sizeof(double) * p_bar, cudaMemcpyDeviceToHost));
    if (d->method_out) CK(cudaMemcpy(d->method_out, ctx->method.get(), sizeof(int) * p_bar, cudaMemcpyDeviceToHost));
    if (d->rank_out) CK(cudaMemcpy(d->rank_out, ctx->rank.get(), sizeof(int) * p_bar, cudaMemcpyDeviceToHost));
    if (d->svd_sweeps_out)
      CK(cudaMemcpy(d->svd_sweeps_out, ctx->sweeps.get(), sizeof(int) * p_bar, cudaMemcpyDeviceToHost));
    if (d->launches_out) *d->launches_out = launches;
    if (phases)
      for (int p = 1; p <= p_bar; ++p) {
        float a = 0.f, b = 0.f, cc = 0.f;
        CK(cudaEventElapsedTime(&a, ctx->events[p - 1], ctx->pev[2 * (p - 1)]));
        CK(cudaEventElapsedTime(&b, ctx->pev[2 * (p - 1)], ctx->pev[2 * (p - 1) + 1]));
        CK(cudaEventElapsedTime(&cc, ctx->pev[2 * (p - 1) + 1], ctx->events[p]));
        d->phase_seconds[3 * (p - 1) + 0] = a * 1e-3;
        d->phase_seconds[3 * (p - 1) + 1] = b * 1e-3;
        d->phase_seconds[3 * (p - 1) + 2] = cc * 1e-3;
      }
  }
}

// ---------------------------------------------------------------------------
// Exact per-lag OLS on the full series (bench.cpp:27-48):
// lag h uses every row i = 0..n-h-1 (forward order y[i .. i + h], target
// last), solved by the same preconditioned CholeskyQR as the sampled systems;
// lag h - 1's factor preconditions lag h (its rows are a superset).

static void exact_sweep(tf_context* ctx, int p_bar, double* taus, double* coefs, double* lag_seconds,
                        int* p_star) {
  if (p_bar < 1) throw TfError{TF_USAGE, "maximum lag must be at least 1"};
  if (ctx->n == 0) throw TfError{TF_USAGE, "no series uploaded"};
  const int64_t n = ctx->n;
  if (n <= (int64_t)p_bar + 1) throw TfError{TF_DATA, "series too short for maximum lag " + std::to_string(p_bar)};
  const int64_t rows_max = n - 1;
  cudaStream_t st = ctx->stream;
  alloc_state(ctx, p_bar, 1, 1);
  ctx->rh_aidx.need(rows_max);
  ctx->rh_ones.need(rows_max);
  k_iota<<<grid_for(rows_max, ctx), 256, 0, st>>>(ctx->rh_aidx.get(), rows_max);
  k_fill<<<grid_for(rows_max, ctx), 256, 0, st>>>(ctx->rh_ones.get(), rows_max, 1.0);
  g_launches += 2;
  reserve_solve(ctx, rows_max, p_bar + 1);
  ctx->rh_rest.need(2);
  ensure_events(ctx, p_bar + 1);
  ensure_span_events(ctx);
  CK(cudaEventRecord(ctx->ev_begin, st));
  CK(cudaEventRecord(ctx->events[0], st));
  for (int h = 1; h <= p_bar; ++h) {
    const int64_t m = n - h;
    SolveOut o;
    o.phi = ctx->phi.get();
    o.coefs = ctx->coefs.get();
    o.coef_off = (int64_t)(h - 1) * h / 2;
    o.taus = ctx->taus.get();
    o.method = ctx->method.get();
    o.lag = h;
    o.status = ctx->status.get();
    FwdRows ld{ctx->y.get(), ctx->rh_aidx.get(), ctx->rh_ones.get(), 0};
    double* Snext = (h & 1) ? ctx->sb.S1.get() : ctx->sb.S0.get();
    const double* Sprev = (h & 1) ? ctx->sb.S0.get() : ctx->sb.S1.get();
    solve_rows(ctx, ld, m, h + 1, o, h >= 2 ? Sprev : nullptr, h >= 2 ? ctx->phi.get() : nullptr, Snext, 0,
               ctx->rh_rest.get(), ctx->rh_rest.get());
    CK(cudaEventRecord(ctx->events[h], st));
  }
  CK(cudaEventRecord(ctx->ev_end, st));
  CK(cudaStreamSynchronize(st));
  int sth[3];
  CK(cudaMemcpy(sth, ctx->status.get(), 3 * sizeof(int), cudaMemcpyDeviceToHost));
  raise_from_status(sth);
  std::vector<double> t(p_bar);
  CK(cudaMemcpy(t.data(), ctx->taus.get(), p_bar * sizeof(double), cudaMemcpyDeviceToHost));
  if (taus) std::memcpy(taus, t.data(), p_bar * sizeof(double));
  if (coefs)
    CK(cudaMemcpy(coefs, ctx->coefs.get(), sizeof(double) * (size_t)p_bar * (p_bar + 1) / 2, cudaMemcpyDeviceToHost));
  if (lag_seconds)
    for (int h = 1; h <= p_bar; ++h) {
      float ms = 0.f;
      CK(cudaEventElapsedTime(&ms, ctx->events[h - 1], ctx->events[h]));
      lag_seconds[h - 1] = ms * 1e-3;
    }
  if (p_star) *p_star = tf_select_order(t.data(), p_bar, 1.96 / std::sqrt((double)(n - p_bar)));
}

// ---------------------------------------------------------------------------
// SRHT sweep (bench.cpp:50-72 srht_fit, sketch.cpp:187-239
// srht_solve): per lag h the signed, zero-padded columns y[i + a] (forward
// order, a = h the target) go through the Walsh-Hadamard transform on the
// device (k_fwht_pass, largest stride first: bit-identical to the reference's
// pruned transform), the c rows below(N) are gathered with weight sqrt(N / c)
// into a dense c x (h + 1) system, and the compressed solve is the LSAR one
// (preconditioned CholeskyQR; lag h - 1's factor preconditions lag h: both
// sketches approximate the same Gram).
// level ranges from the top (largest strides first): 8-level passes while
// at least 12 levels remain (so a strided pass has 16 low offsets), then the
// remainder in one pass
static std::vector<std::pair<int, int>> fwht_passes(int m) {
  std::vector<std::pair<int, int>> ps;
  int rem = m;
  while (rem >= kFwhtLevels + 4) {
    ps.push_back({rem - kFwhtLevels, rem});
    rem -= kFwhtLevels;
  }
  if (rem > 0) ps.push_back({0, rem});
  return ps;
}

static void fwht_columns(tf_context* ctx, double* X, int64_t N, int nb, const double* y, int64_t n0, int a0,
                         uint64_t seed) {
  int m = 0;
  while (((int64_t)1 << m) < N) ++m;
  const auto ps = fwht_passes(m);
  for (size_t k = 0; k < ps.size(); ++k) {
    FwhtArgs a;
    a.X = X;
    a.N = N;
    a.l0 = ps[k].first;
    a.l1 = ps[k].second;
    a.y = k == 0 ? y : nullptr;
    a.n0 = n0;
    a.a0 = a0;
    a.seed = seed;
    const int L = a.l1 - a.l0;
    const int M = 1 << L;
    int LW;  // lanes per CTA (as k_fwht_pass derives them)
    if (L == 8 && (a.l0 == 0 || a.l0 >= 4) && N >= 4096) LW = 16;
    else if (a.l0 == 0) LW = (int)std::min<int64_t>(std::max(1, 4096 / M), N / M);
    else LW = a.l0 >= 4 ? 16 : (1 << a.l0);
    const size_t smem = sizeof(double) * (size_t)M * LW;
    smem_optin((const void*)k_fwht_pass, smem);
    dim3 grid((unsigned)(N / ((int64_t)M * LW)), (unsigned)nb);
    k_fwht_pass<<<grid, kFwhtThreads, smem, ctx->stream>>>(a);
    LAUNCH_CHECK("k_fwht_pass");
    COUNT_LAUNCH();
  }
}

static int64_t bit_ceil64(int64_t v) {
  int64_t n = 1;
  while (n < v) n <<= 1;
  return n;
}

// host below(N) draws (rng.hpp:59-66) for a lag whose device draws hit a rejection
static void srht_host_draws(uint64_t seed, int64_t n0, int64_t N, int64_t c, std::vector<int64_t>& out) {
  const uint64_t limit = 0ull - (uint64_t)N;
  uint64_t t = (uint64_t)n0;
  out.resize(c);
  for (int64_t k = 0; k < c; ++k) {
    uint64_t x;
    do x = rng_draw(seed, t++);
    while (x >= limit);
    out[k] = (int64_t)(x & (uint64_t)(N - 1));
  }
}

static void srht_sweep(tf_context* ctx, int p_bar, int64_t c, uint64_t seed, double* taus, double* coefs,
                       double* lag_seconds, int* p_star) {
  // srht_fit argument checks (bench.cpp:50-56)
  if (p_bar < 1) throw TfError{TF_USAGE, "maximum lag must be at least 1"};
  if (ctx->n == 0) throw TfError{TF_USAGE, "no series uploaded"};
  const int64_t n = ctx->n;
  if (n <= (int64_t)p_bar + 1) throw TfError{TF_DATA, "series too short for maximum lag " + std::to_string(p_bar)};
  if (c < p_bar) throw TfError{TF_USAGE, "sample count below maximum lag"};
  cudaStream_t st = ctx->stream;
  const int Kmax = p_bar + 1;
  const int64_t Nmax = bit_ceil64(n - 1);
  alloc_state(ctx, p_bar, 1, 1);
  reserve_solve(ctx, c, Kmax);
  const int64_t ldD = ldq_of(Kmax);
  ctx->srht_D.need((size_t)c * ldD);
  ctx->srht_draws.need(c);
  ctx->srht_reject.need(p_bar + 1);
  // transform batch: as many columns as fit in ~512 MB
  const int nbmax = (int)std::max<int64_t>(1, std::min<int64_t>(Kmax, ((int64_t)512 << 20) / (Nmax * 8)));
  ctx->srht_X.need((size_t)nbmax * Nmax);
  ctx->rh_rest.need(2);
  ensure_events(ctx, p_bar + 1);
  ensure_span_events(ctx);
  std::vector<int> host_lag(p_bar + 1, 0);  // lags whose device draws hit a rejection
  for (int attempt = 0; attempt < 2; ++attempt) {
    CK(cudaMemsetAsync(ctx->status.get(), 0, 3 * sizeof(int), st));
    CK(cudaMemsetAsync(ctx->srht_reject.get(), 0, sizeof(int) * (p_bar + 1), st));
    CK(cudaEventRecord(ctx->ev_begin, st));
    CK(cudaEventRecord(ctx->events[0], st));
    for (int h = 1; h <= p_bar; ++h) {
      const int64_t n0 = n - h;
      const int64_t N = bit_ceil64(n0);
      const uint64_t sh = derive_seed(seed, (uint64_t)h);
      const int K = h + 1;
      if (host_lag[h]) {
        std::vector<int64_t> dr;
        srht_host_draws(sh, n0, N, c, dr);
        CK(cudaMemcpyAsync(ctx->srht_draws.get(), dr.data(), sizeof(int64_t) * c, cudaMemcpyHostToDevice, st));
        CK(cudaStreamSynchronize(st));
      } else {
        k_srht_draws<<<grid_for(c, ctx), 256, 0, st>>>(sh, n0, N, c, ctx->srht_draws.get(),
                                                       ctx->srht_reject.get() + h);
        LAUNCH_CHECK("k_srht_draws");
        COUNT_LAUNCH();
      }
      const double w = std::sqrt((double)N / (double)c);
      for (int a0 = 0; a0 < K; a0 += nbmax) {
        const int nb = std::min(nbmax, K - a0);
        fwht_columns(ctx, ctx->srht_X.get(), N, nb, ctx->y.get(), n0, a0, sh);
        k_srht_gather<<<grid_for(c * nb, ctx), 256, 0, st>>>(ctx->srht_X.get(), N, nb, ctx->srht_draws.get(), c, w,
                                                            ctx->srht_D.get(), ldD, a0);
        LAUNCH_CHECK("k_srht_gather");
        COUNT_LAUNCH();
      }
      SolveOut o;
      o.phi = ctx->phi.get();
      o.coefs = ctx->coefs.get();
      o.coef_off = (int64_t)(h - 1) * h / 2;
      o.taus = ctx->taus.get();
      o.method = ctx->method.get();
      o.lag = h;
      o.status = ctx->status.get();
      DenseRows ld{ctx->srht_D.get(), ldD};
      double* Snext = (h & 1) ? ctx->sb.S1.get() : ctx->sb.S0.get();
      const double* Sprev = (h & 1) ? ctx->sb.S0.get() : ctx->sb.S1.get();
      solve_rows(ctx, ld, c, K, o, h >= 2 ? Sprev : nullptr, h >= 2 ? ctx->phi.get() : nullptr, Snext, 0,
                 ctx->rh_rest.get(), ctx->rh_rest.get());
      CK(cudaEventRecord(ctx->events[h], st));
    }
    CK(cudaEventRecord(ctx->ev_end, st));
    CK(cudaStreamSynchronize(st));
    std::vector<int> rj(p_bar + 1);
    CK(cudaMemcpy(rj.data(), ctx->srht_reject.get(), sizeof(int) * (p_bar + 1), cudaMemcpyDeviceToHost));
    bool again = false;
    for (int h = 1; h <= p_bar; ++h)
      if (rj[h] && !host_lag[h]) host_lag[h] = 1, again = true;  // below() rejected (p ~ N / 2^64): redo exactly
    if (!again) break;
  }
  int sth[3];
  CK(cudaMemcpy(sth, ctx->status.get(), 3 * sizeof(int), cudaMemcpyDeviceToHost));
  raise_from_status(sth);
  std::vector<double> t(p_bar);
  CK(cudaMemcpy(t.data(), ctx->taus.get(), p_bar * sizeof(double), cudaMemcpyDeviceToHost));
  if (taus) std::memcpy(taus, t.data(), p_bar * sizeof(double));
  if (coefs)
    CK(cudaMemcpy(coefs, ctx->coefs.get(), sizeof(double) * (size_t)p_bar * (p_bar + 1) / 2, cudaMemcpyDeviceToHost));
  if (lag_seconds)
    for (int h = 1; h <= p_bar; ++h) {
      float ms = 0.f;
      CK(cudaEventElapsedTime(&ms, ctx->events[h - 1], ctx->events[h]));
      lag_seconds[h - 1] = ms * 1e-3;
    }
  if (p_star) *p_star = tf_select_order(t.data(), p_bar, 1.96 / std::sqrt((double)c));
}

// orthonormal Walsh-Hadamard transform of a host vector (sketch.cpp:107-120;
// level order largest stride first, as the pruned transform)
static void hadamard_host(tf_context* ctx, double* x, int64_t n) {
  if (n < 1 || (n & (n - 1)) != 0) throw TfError{TF_USAGE, "transform length must be a power of two"};
  cudaStream_t st = ctx->stream;
  ctx->srht_X.need(n);
  CK(cudaMemcpyAsync(ctx->srht_X.get(), x, sizeof(double) * n, cudaMemcpyHostToDevice, st));
  fwht_columns(ctx, ctx->srht_X.get(), n, 1, nullptr, 0, 0, 0);
  CK(cudaMemcpyAsync(x, ctx->srht_X.get(), sizeof(double) * n, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
}

// ---------------------------------------------------------------------------
// On-device synthetic series: cascade of first-order AR
// sections over counter-RNG innovations, written straight into the context's
// series buffer (the generator the BASELINE configs describe; bench inputs of
// C4 size never cross PCIe).
static void generate_series(tf_context* ctx, const double* roots, int q, int64_t n, uint64_t seed,
                            int innovations, int64_t burn_in) {
  if (n < 1 || q < 0 || burn_in < 0) throw TfError{TF_USAGE, "invalid generator arguments"};
  for (int k = 0; k < q; ++k)
    if (!(std::fabs(roots[k]) > 1.0)) throw TfError{TF_USAGE, "AR roots must lie outside the unit circle"};
  cudaStream_t st = ctx->stream;
  const int64_t total = n + burn_in;
  DBuf<double> x;
  x.need(total);
  k_gen_innovations<<<grid_for(total / 2 + 1, ctx), 256, 0, st>>>(seed, total, innovations == 1 ? 1 : 0, x.get());
  LAUNCH_CHECK("k_gen_innovations");
  const int64_t nblk = (total + kGenBlock - 1) / kGenBlock;
  DBuf<double> bend;
  bend.need(nblk);
  for (int k = 0; k < q; ++k) {
    const double a = 1.0 / roots[k];
    double aB = 1.0;
    for (int u = 0; u < kGenBlock; ++u) aB *= a;
    k_ar_scan_local<<<(unsigned)nblk, kGenThreads, 0, st>>>(x.get(), total, a, bend.get());
    k_ar_scan_blocks<<<1, 1024, 0, st>>>(bend.get(), nblk, aB);
    k_ar_scan_apply<<<(unsigned)nblk, kGenThreads, 0, st>>>(x.get(), total, a, bend.get());
    LAUNCH_CHECK("k_ar_scan");
  }
  ctx->y.need(n + 64);
  CK(cudaMemcpyAsync(ctx->y.get(), x.get() + burn_in, n * sizeof(double), cudaMemcpyDeviceToDevice, st));
  CK(cudaMemsetAsync(ctx->y.get() + n, 0, 64 * sizeof(double), st));
  CK(cudaStreamSynchronize(st));
  x.release();
  bend.release();
  ctx->n = n;
}

static void download_series(tf_context* ctx, double* out, int64_t n) {
  CK(cudaMemcpyAsync(out, ctx->y.get(), n * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
}

__global__ void __launch_bounds__(256) k_dfma_probe(double* out, int iters, double seed) {
  double a0 = seed + threadIdx.x, a1 = a0 * 0.5, a2 = a0 * 0.25, a3 = a0 * 0.125;
  double a4 = a0 + 1, a5 = a1 + 1, a6 = a2 + 1, a7 = a3 + 1;
  const double m = 0.999999999, c = 1e-9;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      a0 = fma(a0, m, c); a1 = fma(a1, m, c); a2 = fma(a2, m, c); a3 = fma(a3, m, c);
      a4 = fma(a4, m, c); a5 = fma(a5, m, c); a6 = fma(a6, m, c); a7 = fma(a7, m, c);
    }
  }
  const double r = ((a0 + a1) + (a2 + a3)) + ((a4 + a5) + (a6 + a7));
  if (r == 12345.678) out[threadIdx.x] = r;
}

static double probe_fp64(tf_context* ctx) {
  DBuf<double> out;
  out.need(256);
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  const int blocks = ctx->sm_count * 8, iters = 4096;
  k_dfma_probe<<<blocks, 256, 0, ctx->stream>>>(out.get(), 64, 1.0);  // warm-up
  CK(cudaEventRecord(e0, ctx->stream));
  k_dfma_probe<<<blocks, 256, 0, ctx->stream>>>(out.get(), iters, 1.0);
  CK(cudaEventRecord(e1, ctx->stream));
  CK(cudaEventSynchronize(e1));
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  out.release();
  const double flops = 2.0 * 8 * 16 * (double)iters * 256 * blocks;
  return flops / (ms * 1e-3) / 1e12;
}

}  // namespace tfe

// ===========================================================================
// C ABI
// ===========================================================================
using tfe::TfError;

template <class F>
static tf_status guarded(tf_context* ctx, F&& f) {
  try {
    f();
    if (ctx) ctx->err.clear();
    return TF_OK;
  } catch (const TfError& e) {
    if (ctx) ctx->err = e.msg;
    return e.code;
  } catch (const std::bad_alloc&) {
    if (ctx) ctx->err = "host allocation failed";
    return TF_CUDA;
  }
}

extern "C" {

const char* tf_version(void) { return "toepfit-b200 0.1 (sm_100a)"; }

tf_status tf_create(const tf_opts* opts, tf_context** out) {
  if (!out) return TF_USAGE;
  *out = nullptr;
  int dev = opts ? opts->device : 0;
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) return TF_CUDA;
  if (dev < 0 || dev >= count) return TF_USAGE;
  if (cudaSetDevice(dev) != cudaSuccess) return TF_CUDA;
  tf_context* ctx = new (std::nothrow) tf_context();
  if (!ctx) return TF_CUDA;
  ctx->device = dev;
  cudaDeviceGetAttribute(&ctx->sm_count, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&ctx->smem_optin_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  {
    const char* v = std::getenv("TF_NO_GRAPHS");  // debugging: launch every sweep eagerly
    ctx->no_graphs = v && v[0] == '1';
    const char* gm = std::getenv("TF_GRAM");  // "dd" / "i8": force one Gram path (parity tests, benchmarks)
    ctx->gram_mode = gm && !std::strcmp(gm, "dd") ? 1 : gm && !std::strcmp(gm, "i8") ? 2 : 0;
    const char* pm = std::getenv("TF_PASS");  // "dmma" / "fft": force one pass path (parity tests, benchmarks)
    ctx->pass_mode = pm && !std::strcmp(pm, "dmma") ? 1 : pm && !std::strcmp(pm, "fft") ? 2 : 0;
    const char* mq = std::getenv("TF_FFT_MINQ");  // crossover lag of the auto mode
    ctx->fft_minq = mq ? std::max(1, std::atoi(mq)) : tfe::kFftMinQ;
    ctx->fft_minlags = mq ? 0 : tfe::kFftMinLags;  // a forced crossover is taken as given
    const char* sp = std::getenv("TF_FFT_SPLIT");  // 0: the score update stays fused into the FFT pass
    ctx->fft_split = sp ? std::atoi(sp) != 0 : 1;
    const char* fs = std::getenv("TF_FFT_SLOTS");  // deferred-folding groups of the FFT pass (1..4)
    ctx->fft_slots = fs ? std::min(tfk::kFftSlots, std::max(1, std::atoi(fs))) : tfk::kFftSlots;
  }
  int least = 0, greatest = 0;
  cudaDeviceGetStreamPriorityRange(&least, &greatest);
  const int prio = std::max(greatest, least - std::max(0, opts ? opts->priority : 0));
  // the side stream (the FFT lags' score updates beside the solve) sits one priority step below the
  // main one, so the solve's kernels take the SMs as soon as they are launched
  const int main_prio = std::max(greatest, prio - 1);  // k levels above the default keeps its meaning
  if (cudaStreamCreateWithPriority(&ctx->stream, cudaStreamNonBlocking, main_prio) != cudaSuccess) {
    delete ctx;
    return TF_CUDA;
  }
  if (cudaStreamCreateWithPriority(&ctx->side, cudaStreamNonBlocking, least) != cudaSuccess ||
      cudaEventCreateWithFlags(&ctx->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&ctx->ev_join, cudaEventDisableTiming) != cudaSuccess) {
    cudaStreamDestroy(ctx->stream);
    delete ctx;
    return TF_CUDA;
  }
  *out = ctx;
  return TF_OK;
}

void tf_destroy(tf_context* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  for (auto e : ctx->events) cudaEventDestroy(e);
  for (auto e : ctx->pev) cudaEventDestroy(e);
  if (ctx->ev_begin) cudaEventDestroy(ctx->ev_begin);
  if (ctx->ev_end) cudaEventDestroy(ctx->ev_end);
  if (ctx->lsar_graph.exec) cudaGraphExecDestroy(ctx->lsar_graph.exec);
  if (ctx->rh_graph.exec) cudaGraphExecDestroy(ctx->rh_graph.exec);
  if (ctx->comm) ncclCommDestroy(ctx->comm);
  if (ctx->side) {
    cudaStreamSynchronize(ctx->side);
    cudaStreamDestroy(ctx->side);
  }
  if (ctx->ev_fork) cudaEventDestroy(ctx->ev_fork);
  if (ctx->ev_join) cudaEventDestroy(ctx->ev_join);
  cudaStreamDestroy(ctx->stream);
  delete ctx;  // DBuf destructors free every device buffer
}

const char* tf_last_error(const tf_context* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

tf_status tf_upload_series(tf_context* ctx, const double* y, int64_t n) {
  if (!ctx) return TF_USAGE;
  return guarded(ctx, [&] {
    cudaSetDevice(ctx->device);
    tfe::upload_series(ctx, y, n, false);
  });
}

tf_status tf_upload_series_device(tf_context* ctx, const double* d_y, int64_t n) {
  if (!ctx) return TF_USAGE;
  return guarded(ctx, [&] {
    cudaSetDevice(ctx->device);
    tfe::upload_series(ctx, d_y, n, true);
  });
}

tf_status tf_lsar_sweep(tf_context* ctx, int p_bar, int64_t c, uint64_t seed, const tf_lsar_diag* diag,
                        double* taus, double* coefs_packed, double* lag_seconds, int* p_star) {
  if (!ctx) return TF_USAGE;
  return guarded(ctx, [&] {
    cudaSetDevice(ctx->device);
    tfe::lsar_sweep(ctx, p_bar, c, seed, diag, taus, coefs_packed, lag_seconds, p_star);
  });
}

tf_status tf_lsar_sweep_batch(tf_context* ctx, const double* y, int64_t y_stride, int64_t batch, int64_t n,
                              int p_bar, int64_t c, const uint64_t* seeds, const int64_t* fixed_idx,
                              const double* fixed_w, double* taus, double* coefs_packed, double* lag_seconds,
                              int* p_star, int* status_out) {
  if (!ctx || !y || !seeds || batch < 1) return TF_USAGE;
  return guarded(ctx, [&] {
    cudaSetDevice(ctx->device);
    const int64_t ncoef = (int64_t)p_bar * (p_bar + 1) / 2;
    std::vector<double> t((size_t)(batch * std::max(p_bar, 1))), cf((size_t)(batch * std::max<int64_t>(ncoef, 1)));
    std::vector<int> stv((size_t)(3 * batch)), fb((size_t)batch);
    tfe::lsar_batch(ctx, y, y_stride, batch, n, p_bar, c, seeds, fixed_idx, fixed_w, t.data(), cf.data(),
                    lag_seconds, stv.data(), fb.data());
    // series whose sampled system broke down: the single-series path (shifted
    // CholeskyQR3 / minimum-norm answers, tf_lsar_sweep)
    for (int64_t b = 0; b < batch; ++b) {
      if (!fb[b]) continue;  // (a flagged fit's later lags ran on stale state: its status is moot)
      stv[3 * b] = stv[3 * b + 1] = stv[3 * b + 2] = 0;
      tfe::upload_series(ctx, y + b * y_stride, n, false);
      tf_lsar_diag d{};
      if (fixed_idx && fixed_w) {
        d.fixed_idx = fixed_idx + b * p_bar * c;
        d.fixed_w = fixed_w + b * p_bar * c;
      }
      try {
        tfe::lsar_sweep(ctx, p_bar, c, seeds[b], (fixed_idx && fixed_w) ? &d : nullptr, t.data() + b * p_bar,
                        cf.data() + b * ncoef, nullptr, nullptr);
      } catch (const tfe::TfError& e) {
        stv[3 * b] = e.code == TF_USAGE ? kErrUsage : e.code == TF_DATA ? kErrData : kErrNumerical;
        stv[3 * b + 2] = kReasonCholFail;
      }
    }
    for (int64_t b = 0; b < batch; ++b) {
      if (taus) std::memcpy(taus + b * p_bar, t.data() + b * p_bar, p_bar * sizeof(double));
      if (coefs_packed) std::memcpy(coefs_packed + b * ncoef, cf.data() + b * ncoef, ncoef * sizeof(double));
      if (p_star) p_star[b] = stv[3 * b] ? 0 : tf_select_order(t.data() + b * p_bar, p_bar, 1.96 / std::sqrt((double)c));
      if (status_out)
        for (int k = 0; k < 3; ++k) status_out[3 * b + k] = stv[3 * b + k];
    }
  });
}

tf_status tf_generalized_leverage(tf_context* ctx, const double* c_rows, int64_t rows, int64_t c_cols, const double* b,
                                  int64_t brows, int64_t b_cols, int64_t sketch_rows, uint64_t sketch_seed, double* out) {
  if (!ctx || (rows > 0 && (!c_rows || !out)) || (brows > 0 && !b)) return TF_USAGE;
  return guarded(ctx, [&] {
    cudaSetDevice(ctx->device);
    tfe::generalized_leverage(ctx, c_rows, rows, c_cols, b, brows, b_cols, sketch_rows, sketch_seed, out);
  });
}

tf_status tf_repeated_halving(tf_context* ctx, int64_t n, int64_t k, tf_gather_fn gather, void* user,
                              const tf_rh_cfg* cfg, double* approx_out, int64_t approx_cap, int64_t* approx_rows,
                              int* levels) {
  if (!ctx || !approx_out) return TF_USAGE;
  return guarded(ctx, [&] {
    cudaSetDevice(ctx->device);
    tfe::repeated_halving_src(ctx, n, k, gather, user, cfg, approx_out, approx_cap, approx_rows, levels);
  });
}

tf_status tf_lsar_step(tf_context* ctx, int p_bar, int64_t c, uint64_t seed, int p, const double* scores_in,
                       const double* resid_in, double* scores_out, double* resid_out, double* phi_out, int* method_out) {
  if (!ctx) return TF_USAGE;
  return guarded(ctx, [&] {
    cudaSetDevice(ctx->device);
    tfe::lsar_step(ctx, p_bar, c, seed, p, scores_in, resid_in, scores_out, resid_out, phi_out, method_out);
  });
}

tf_status tf_residuals(tf_context* ctx, const double* y, int64_t n_used, int p, const double* phi,
                       double* r_out) {
  if (!ctx) return TF_USAGE;
  return guarded(ctx, [&] { tfe::residuals_op(ctx, y, n_used, p, phi, r_out); });
}

tf_status tf_sample_rows(tf_context* ctx, const double* scores, int64_t n, int64_t c, uint64_t seed,
                         int64_t* idx_out, double* w_out) {
  if (!ctx) return TF_USAGE;
  return guarded(ctx, [&] { tfe::sample_op(ctx, scores, n, c, seed, idx_out, w_out); });
}

tf_status tf_apply_sample(tf_context* ctx, const double* y, int64_t n_used, int p, const int64_t* idx,
                          const double* w, int64_t c, int width, double* a_out, double* b_out) {
  if (!ctx) return TF_USAGE;
  return guarded(ctx, [&] { tfe::apply_sample_op(ctx, y, n_used, p, idx, w, c, width, a_out, b_out); });
}

tf_status tf_solve_sampled(tf_context* ctx, const double* y, int64_t n_used, int p, const int64_t* idx,
                           const double* w, int64_t c, double* phi_out, int* method_out) {
  if (!ctx) return TF_USAGE;
  return guarded(ctx, [&] { tfe::solve_sampled_op(ctx, y, n_used, p, idx, w, c, phi_out, method_out); });
}

tf_status tf_rh_sweep(tf_context* ctx, int p_bar, int64_t c, const tf_rh_cfg* cfg, uint64_t seed,
                      const tf_rh_diag* diag, double* taus, double* coefs_packed,
                      double* lag_seconds, double* upfront_seconds, int* p_star) {
  if (!ctx) return TF_USAGE;
  return guarded(ctx, [&] {
    cudaSetDevice(ctx->device);
    tfe::rh_sweep(ctx, p_bar, c, cfg, seed, diag, taus, coefs_packed, lag_seconds, upfront_seconds,
                  p_star);
  });
}

int tf_select_order(const double* taus, int p_bar, double bound) {
  // toeplitz.cpp:133-138: largest lag whose |tau| clears the bound (inclusive)
  for (int h = p_bar; h >= 1; --h)
    if (std::fabs(taus[h - 1]) >= bound) return h;
  return 0;
}

uint64_t tf_derive_seed(uint64_t seed, uint64_t tag) { return tfk::derive_seed(seed, tag); }

tf_status tf_exact_sweep(tf_context* ctx, int p_bar, double* taus, double* coefs_packed, double* lag_seconds,
                         int* p_star) {
  if (!ctx) return TF_USAGE;
  return guarded(ctx, [&] { tfe::exact_sweep(ctx, p_bar, taus, coefs_packed, lag_seconds, p_star); });
}

tf_status tf_srht_sweep(tf_context* ctx, int p_bar, int64_t c, uint64_t seed, double* taus, double* coefs_packed,
                        double* lag_seconds, int* p_star) {
  if (!ctx) return TF_USAGE;
  return guarded(ctx, [&] { tfe::srht_sweep(ctx, p_bar, c, seed, taus, coefs_packed, lag_seconds, p_star); });
}

tf_status tf_hadamard(tf_context* ctx, double* x, int64_t n) {
  if (!ctx || !x) return TF_USAGE;
  return guarded(ctx, [&] { tfe::hadamard_host(ctx, x, n); });
}

tf_status tf_download_series(tf_context* ctx, double* out, int64_t n) {
  if (!ctx || !out || n < 0 || n > ctx->n) return TF_USAGE;
  return guarded(ctx, [&] { tfe::download_series(ctx, out, n); });
}

tf_status tf_generate_series(tf_context* ctx, const double* roots, int q, int64_t n, uint64_t seed,
                             int innovations, int64_t burn_in) {
  if (!ctx || (q > 0 && !roots)) return TF_USAGE;
  return guarded(ctx, [&] { tfe::generate_series(ctx, roots, q, n, seed, innovations, burn_in); });
}

tf_status tf_sweep_span(const tf_context* ref, const tf_context* ctx, double* start_ms, double* end_ms) {
  if (!ref || !ctx || !start_ms || !end_ms || !ref->ev_begin || !ctx->ev_begin || !ctx->ev_end) return TF_USAGE;
  float a = 0.f, b = 0.f;
  if (cudaEventElapsedTime(&a, ref->ev_begin, ctx->ev_begin) != cudaSuccess) return TF_CUDA;
  if (cudaEventElapsedTime(&b, ref->ev_begin, ctx->ev_end) != cudaSuccess) return TF_CUDA;
  *start_ms = a;
  *end_ms = b;
  return TF_OK;
}

tf_status tf_nccl_unique_id(unsigned char* out, int bytes) {
  if (!out || bytes < (int)sizeof(ncclUniqueId)) return TF_USAGE;
  ncclUniqueId uid;
  if (ncclGetUniqueId(&uid) != ncclSuccess) return TF_NCCL;
  std::memcpy(out, &uid, sizeof uid);
  return TF_OK;
}

tf_status tf_nccl_init(tf_context* ctx, const unsigned char* id, int world, int rank) {
  if (!ctx || !id) return TF_USAGE;
  return guarded(ctx, [&] {
    cudaSetDevice(ctx->device);
    tfe::nccl_init(ctx, id, world, rank);
  });
}

tf_status tf_keep_slice(tf_context* ctx, int64_t start, int64_t len) {
  if (!ctx) return TF_USAGE;
  return guarded(ctx, [&] {
    cudaSetDevice(ctx->device);
    tfe::keep_slice(ctx, start, len);
  });
}

tf_status tf_lsar_sweep_sharded(tf_context* ctx, int p_bar, int64_t c, uint64_t seed, const tf_lsar_diag* diag,
                                double* taus, double* coefs_packed, double* lag_seconds, int* p_star) {
  if (!ctx) return TF_USAGE;
  return guarded(ctx, [&] {
    cudaSetDevice(ctx->device);
    tfe::lsar_sweep_sharded(ctx, p_bar, c, seed, diag, taus, coefs_packed, lag_seconds, p_star);
  });
}

int64_t tf_tpu_size(int K) { return K < 1 ? 0 : tfk::tpu_size(K); }

tf_status tf_fft_first_lag(tf_context* ctx, int p_bar, int* lag) {
  if (!ctx || !lag || p_bar < 1) return TF_USAGE;
  int q = 1;
  while (q <= p_bar && !tfe::fft_lag(ctx, p_bar, q)) ++q;
  *lag = q;
  return TF_OK;
}

tf_status tf_probe_fp64_peak(tf_context* ctx, double* tflops) {
  if (!ctx || !tflops) return TF_USAGE;
  return guarded(ctx, [&] {
    cudaSetDevice(ctx->device);
    *tflops = tfe::probe_fp64(ctx);
  });
}

}  // extern "C"
