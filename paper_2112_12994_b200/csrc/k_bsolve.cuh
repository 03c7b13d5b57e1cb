// k_bsolve.cuh -- the per-lag sampled solve of a BATCH of small LSAR systems
// (K = p + 1 <= 64, any c), one CTA per series (replaces, per series, the
// Eigen ColPivHouseholderQR of toeplitz.cpp:57-71 behind solve_compressed,
// sketch.cpp:96-101, as the single-series path's k_qform / k_gram / k_cholinv
// / k_phi_solve chain does -- but in one launch for all series of the batch).
//
// Same method as the single-series path (DESIGN 4.2): preconditioned
// CholeskyQR.  With the previous lag's composite factor S_{p-1} and phi_{p-1},
//   T = [[S_{p-1}, u], [0, 1/s]],  u = -(0, phi_fwd_{p-1}) / s,  s = ||r_{p-1}||
// (k_precond), M := T; pass A: G = (A M)^T (A M), R = chol(G), M := M R^-1;
// pass B (gated: ||R||_F ||R^-1||_F > 8 K) repeats with the new M.  The rows
// of A are w_t y[i_t + a], a = 0..p (forward order, target last), gathered in
// 32-row chunks; A M and the Gram are formed in fp64 on the CUDA cores (a
// K <= 64 system leaves nothing for the tensor cores to amortise).
//   phi_fwd = -v[0..p) / v[p],  v = M e_p  (the last column of M: A v is the
//   residual direction, orthogonal to the lag columns);  phi[j] = phi_fwd[p-1-j]
// M is the next lag's S.  A Cholesky breakdown (rank-deficient sample) sets
// the series' fallback flag: the host re-runs that series through the
// single-series path, which has the shifted / minimum-norm answers.
#pragma once

#include "common.cuh"

namespace tfk {

constexpr int kBsMaxK = 64;
constexpr int kBsLd = 66;     // shared row stride (doubles): 16-byte rows, spread banks
constexpr int kBsALd = 65;    // gathered chunk rows: odd stride, lane-per-row reads conflict free
constexpr int kBsCh = 32;     // rows per gathered chunk
constexpr int kBsThreads = 256;
constexpr int kBsSLd = 64;    // global S stride (dense K x K per series)

struct BSolveArgs {
  const double* y;        // series b at y + b * bs_y
  int64_t bs_y;
  const int64_t* idx;     // draws of series b at idx + b * bs_idx (this lag's c rows)
  const double* wts;
  int64_t bs_idx;
  int64_t c;
  int K;                  // p + 1
  int lag;                // p
  const double* Sprev;    // lag p-1's M (dense, ld kBsSLd), series stride kBsSLd^2
  double* Snext;
  double* phi;            // in: phi_{p-1}; out: phi_p (stride bs_phi)
  int64_t bs_phi;
  const double* scal;     // 4 per series: scal[0] = R_{p-1}
  double* coefs;          // packed p_bar (p_bar + 1) / 2 per series
  int64_t bs_coef;
  double* taus;           // p_bar per series
  int64_t bs_tau;
  int* method;            // p_bar per series
  int* fallback;          // 1 per series
};

__host__ inline size_t bsolve_smem_bytes() {
  return sizeof(double) * (size_t)(3 * kBsMaxK * kBsLd);
}

__global__ void __launch_bounds__(kBsThreads, 2) k_bsolve(BSolveArgs a) {
  extern __shared__ __align__(16) double bsm[];
  // rows of kBsLd doubles: Ms [0, 64); chunk phase: A buffers [64, 96) and
  // [96, 128), Q [128, 160); factor phase: Gs [64, 128), R^-1 [128, 192)
  double* Ms = bsm;                       // composite right factor M (upper)
  double* Gs = Ms + kBsMaxK * kBsLd;      // Gram -> R (upper), then M R^-1
  double* Ab = Gs;                        // two chunk buffers (cp.async targets)
  double* Qs = Gs + 2 * kBsCh * kBsLd;
  double* Ri = Gs + kBsMaxK * kBsLd;
  __shared__ int64_t sIdx[3][kBsCh];      // row offsets / weights, two chunks ahead
  __shared__ double sW[3][kBsCh];
  const int64_t b = blockIdx.x;
  const int tid = threadIdx.x;
  const int K = a.K, p = K - 1;
  const int64_t c = a.c;
  const double* y = a.y + b * a.bs_y;
  const int64_t* idx = a.idx + b * a.bs_idx;
  const double* wt = a.wts + b * a.bs_idx;
  double* phi = a.phi + b * a.bs_phi;
  if (a.fallback[b]) return;  // an earlier lag already sent this series to the single path
  __shared__ int s_flag;
  __shared__ double s_val[2];

  // ---- T (k_precond) into Ms; identity for p = 1 ----
  {
    const double s = sqrt(fmax(a.scal[4 * b], 1e-300));
    const double inv_s = 1.0 / s;
    const double* Sp = a.Sprev + b * (int64_t)kBsSLd * kBsSLd;
    for (int e = tid; e < kBsMaxK * kBsLd; e += kBsThreads) Ms[e] = 0.0;  // columns >= K stay 0
    __syncthreads();
    for (int e = tid; e < K * K; e += kBsThreads) {
      const int r = e / K, cc = e - r * K;
      double v = 0.0;
      if (p == 1) v = r == cc ? 1.0 : 0.0;
      else if (r <= cc) {
        if (cc < p) v = Sp[r * kBsSLd + cc];
        else if (r == p) v = inv_s;
        else v = r == 0 ? 0.0 : -phi[p - 1 - r] * inv_s;
      }
      Ms[r * kBsLd + cc] = v;
    }
  }
  // register-blocked Gram: the upper 4 x 4 blocks (bi <= bj) of G, two
  // threads per block (even / odd chunk rows) while they fit in the CTA
  const int nb4 = (K + 3) >> 2, nblk = nb4 * (nb4 + 1) / 2;
  const int split = 2 * nblk <= kBsThreads ? 2 : 1;
  const int gtask = tid / split, ghalf = tid % split;
  int bi = 0, bj = 0;
  const bool gact = gtask < nblk;
  if (gact) {  // row-major enumeration of the upper blocks
    int rem = gtask;
    while (rem >= nb4 - bi) {
      rem -= nb4 - bi;
      ++bi;
    }
    bj = bi + rem;
  }
  const int lane = tid & 31, warp = tid >> 5;
  const int nch = (int)((c + kBsCh - 1) / kBsCh);
  int passes = 0, need_b = (p == 1);
  for (int pass = 0; pass < 2; ++pass) {
    __syncthreads();
    double g[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) g[i][j] = 0.0;
    // Chunk pipeline: the 32 gathered rows of chunk ch + 1 stream into the
    // other A buffer with 8-byte cp.async (zero fill past K / c) while chunk
    // ch is multiplied; their row offsets and weights were read two chunks
    // ahead into shared memory.  A row's weight scales its Q row after the
    // product (as k_qform_pipe does), so loaded values are never consumed in
    // registers.
    auto load_idx = [&](int ch, int slot) {  // threads 0..31
      const int64_t t = (int64_t)ch * kBsCh + tid;
      sIdx[slot][tid] = t < c ? idx[t] : -1;
      sW[slot][tid] = t < c ? wt[t] : 0.0;
    };
    auto issue = [&](int ch) {
      double* dst = Ab + (ch & 1) * kBsCh * kBsALd;
      const int slot = ch % 3;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int e = tid + kBsThreads * u, r = e >> 6, k = e & 63;
        const int64_t off = sIdx[slot][r];
        const bool ok = off >= 0 && k < K;
        const unsigned d = (unsigned)__cvta_generic_to_shared(dst + r * kBsALd + k);
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(d), "l"(ok ? y + off + k : y),
                     "r"(ok ? 8 : 0)
                     : "memory");
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
    if (tid < kBsCh) {
      load_idx(0, 0);
      if (nch > 1) load_idx(1, 1);
    }
    __syncthreads();
    issue(0);
    for (int ch = 0; ch < nch; ++ch) {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
      __syncthreads();  // chunk ch landed (every thread's copies); Q free
      if (ch + 1 < nch) issue(ch + 1);
      int64_t nidx = -1;
      double nw = 0.0;
      if (tid < kBsCh && ch + 2 < nch) {  // consumed only after the multiply
        const int64_t t = (int64_t)(ch + 2) * kBsCh + tid;
        nidx = t < c ? idx[t] : -1;
        nw = t < c ? wt[t] : 0.0;
      }
      // Q = diag(w) (Y M) for the chunk (32 x K): lane = chunk row, warp w
      // takes column groups w and 15 - w (4 columns each; the triangular
      // depths of the pair sum to a constant, and every lane of a warp runs
      // the same depth -- no divergence)
      const double* As = Ab + (ch & 1) * kBsCh * kBsALd;
      {
        const double* arow = As + lane * kBsALd;
        const double wr = sW[ch % 3][lane];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int cg = h ? 15 - warp : warp;
          if (4 * cg >= K) continue;
          const int qk = min(K, 4 * cg + 4);  // M upper: rows k <= column
          double q[4] = {0.0, 0.0, 0.0, 0.0};
          for (int k = 0; k < qk; ++k) {
            const double2 m01 = *reinterpret_cast<const double2*>(Ms + k * kBsLd + 4 * cg);
            const double2 m23 = *reinterpret_cast<const double2*>(Ms + k * kBsLd + 4 * cg + 2);
            const double x = arow[k];
            q[0] = fma(x, m01.x, q[0]);
            q[1] = fma(x, m01.y, q[1]);
            q[2] = fma(x, m23.x, q[2]);
            q[3] = fma(x, m23.y, q[3]);
          }
          *reinterpret_cast<double2*>(Qs + lane * kBsLd + 4 * cg) = make_double2(wr * q[0], wr * q[1]);
          *reinterpret_cast<double2*>(Qs + lane * kBsLd + 4 * cg + 2) = make_double2(wr * q[2], wr * q[3]);
        }
      }
      __syncthreads();
      if (gact) {
        for (int r = ghalf; r < kBsCh; r += split) {
          const double2 u01 = *reinterpret_cast<const double2*>(Qs + r * kBsLd + 4 * bi);
          const double2 u23 = *reinterpret_cast<const double2*>(Qs + r * kBsLd + 4 * bi + 2);
          const double2 v01 = *reinterpret_cast<const double2*>(Qs + r * kBsLd + 4 * bj);
          const double2 v23 = *reinterpret_cast<const double2*>(Qs + r * kBsLd + 4 * bj + 2);
          const double uu[4] = {u01.x, u01.y, u23.x, u23.y}, vv[4] = {v01.x, v01.y, v23.x, v23.y};
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) g[i][j] = fma(uu[i], vv[j], g[i][j]);
        }
      }
      if (tid < kBsCh && ch + 2 < nch) {
        sIdx[(ch + 2) % 3][tid] = nidx;
        sW[(ch + 2) % 3][tid] = nw;
      }
    }
    __syncthreads();
    // G = sum of the row-half partials (half 0 + half 1, fixed order)
    if (gact && ghalf == 1) {
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) Ri[(4 * bi + i) * kBsLd + 4 * bj + j] = g[i][j];
    }
    __syncthreads();
    if (gact && ghalf == 0) {
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int r = 4 * bi + i, cc = 4 * bj + j;
          const double v = split == 2 ? g[i][j] + Ri[r * kBsLd + cc] : g[i][j];
          if (r < K && cc < K && r <= cc) Gs[r * kBsLd + cc] = v;
        }
    }
    __syncthreads();
    ++passes;
    // ---- p = 1: phi = g01 / g00 (k_solve_k2; exact for the geometric series) ----
    if (p == 1) {
      if (tid == 0) {
        const double g00 = Gs[0], g01 = Gs[1], g11 = Gs[kBsLd + 1];
        const double ph = g01 / g00;
        phi[0] = ph;
        a.coefs[b * a.bs_coef] = ph;
        a.taus[b * a.bs_tau] = ph;
        a.method[b * a.bs_tau] = 0;
        const double r00 = sqrt(g00), r01 = g01 / r00;
        double piv = g11 - r01 * r01;
        const double floor = 4.930380657631324e-32 * (g00 + g11);
        if (!(piv > floor)) piv = floor;
        const double r11 = sqrt(piv);
        double* Sn = a.Snext + b * (int64_t)kBsSLd * kBsSLd;
        Sn[0] = 1.0 / r00;
        Sn[1] = -r01 / (r00 * r11);
        Sn[kBsSLd] = 0.0;
        Sn[kBsSLd + 1] = 1.0 / r11;
      }
      return;
    }
    // ---- Cholesky G = R^T R in place (upper), breakdown -> fallback ----
    if (tid < 32) {
      double tr = 0.0;
      for (int i = tid; i < K; i += 32) tr += Gs[i * kBsLd + i];
      tr = warp_sum(tr);
      if (tid == 0) {
        s_val[0] = (double)max(c, (int64_t)K) * 2.220446049250313e-16 * tr;  // pivot floor
        s_val[1] = tr;
        s_flag = 0;
      }
    }
    __syncthreads();
    const double pfloor = s_val[0];
    for (int k = 0; k < K; ++k) {
      const double d = Gs[k * kBsLd + k];
      if (!(d > pfloor)) {  // uniform: every thread reads the same pivot
        if (tid == 0) a.fallback[b] = 1;
        return;
      }
      const double rkk = sqrt(d), inv = 1.0 / rkk;
      __syncthreads();  // every thread has read the pivot
      if (tid == 0) Gs[k * kBsLd + k] = rkk;
      for (int j = k + 1 + tid; j < K; j += kBsThreads) Gs[k * kBsLd + j] *= inv;
      __syncthreads();
      const int m = K - k - 1;
      for (int e = tid; e < m * m; e += kBsThreads) {
        const int i = k + 1 + e / m, j = k + 1 + e % m;
        if (i <= j) Gs[i * kBsLd + j] = fma(-Gs[k * kBsLd + i], Gs[k * kBsLd + j], Gs[i * kBsLd + j]);
      }
      __syncthreads();
    }
    // ---- R^-1 (upper) into the chunk scratch, column j by thread j ----
    if (tid < K) {
      const int j = tid;
      for (int i = K - 1; i >= 0; --i) {
        double v = (i == j) ? 1.0 : 0.0;
        if (i < j) {
          v = 0.0;
          for (int k = i + 1; k <= j; ++k) v = fma(-Gs[i * kBsLd + k], Ri[k * kBsLd + j], v);
        }
        Ri[i * kBsLd + j] = i <= j ? v / Gs[i * kBsLd + i] : 0.0;
      }
    }
    __syncthreads();
    // gate (pass A): ||R||_F ||R^-1||_F > 8 K -> pass B
    if (pass == 0 && tid < 32) {
      double fr = 0.0, fi = 0.0;
      for (int e = tid; e < K * K; e += 32) {
        const int i = e / K, j = e - i * K;
        if (i <= j) {
          const double x = Gs[i * kBsLd + j], z = Ri[i * kBsLd + j];
          fr = fma(x, x, fr);
          fi = fma(z, z, fi);
        }
      }
      fr = warp_sum(fr);
      fi = warp_sum(fi);
      if (tid == 0) s_flag = (need_b || !(sqrt(fr * fi) <= 8.0 * K)) ? 1 : 0;
    }
    __syncthreads();
    // M := M R^-1 (both upper) into Gs, then back to Ms
    for (int e = tid; e < K * K; e += kBsThreads) {
      const int i = e / K, j = e - i * K;
      double v = 0.0;
      if (i <= j)
        for (int k = i; k <= j; ++k) v = fma(Ms[i * kBsLd + k], Ri[k * kBsLd + j], v);
      Gs[i * kBsLd + j] = v;
    }
    __syncthreads();
    for (int e = tid; e < K * K; e += kBsThreads) {
      const int i = e / K, j = e - i * K;
      Ms[i * kBsLd + j] = Gs[i * kBsLd + j];
    }
    need_b = s_flag;
    if (pass == 0 && !need_b) break;
  }
  __syncthreads();
  // ---- phi from the last column of M; M is the next lag's S ----
  const double vp = Ms[p * kBsLd + p];
  for (int j = tid; j < p; j += kBsThreads) {
    const double ph = -Ms[(p - 1 - j) * kBsLd + p] / vp;
    phi[j] = ph;
    a.coefs[b * a.bs_coef + (int64_t)(p - 1) * p / 2 + j] = ph;
    if (j == p - 1) a.taus[b * a.bs_tau + p - 1] = ph;
  }
  if (tid == 0) a.method[b * a.bs_tau + p - 1] = passes;
  double* Sn = a.Snext + b * (int64_t)kBsSLd * kBsSLd;
  for (int e = tid; e < K * K; e += kBsThreads) {
    const int i = e / K, j = e - i * K;
    Sn[i * kBsSLd + j] = Ms[i * kBsLd + j];
  }
}

}  // namespace tfk
