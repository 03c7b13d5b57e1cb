// k_tpu.cuh -- "tile-packed upper" (TPU) storage and the small kernels of the
// preconditioned CholeskyQR solve.
//
// Column order.  Every sampled least-squares system is handled in *forward*
// order: row t of the lag-p system is the contiguous slice
//     a_t = w_t * (y[b_t], y[b_t + 1], ..., y[b_t + p])     (b_t = i_t + off)
// whose last entry is the target (toeplitz.hpp:29-31 with the columns
// reversed).  In this order the lag-(p-1) augmented matrix is exactly the
// leading p columns of the lag-p one, so the inverse factor S_{p-1} =
// R_{p-1}^-1 of the previous lag preconditions the next lag (sketch-and-
// precondition across lags):
//     T_p = [ S_{p-1}   u ]     u = -(0, phi_{p-1} shifted) / s,  s = ||r_{p-1}||
//           [   0     1/s ]
// Q1 = A T_p is then close to orthonormal and a single CholeskyQR pass is
// usually enough (a second/third pass is gated on the measured conditioning
// or a breakdown).  phi = R_A^-1 z is read off S_p = T_p Rinv_A Rinv_B ...:
//     phi_fwd = -S_p[:p, p] / S_p[p, p],  phi[j] = phi_fwd[p-1-j].
//
// TPU layout of an upper-triangular K x K matrix: 32 x 32 tiles (I <= J),
// each column-major with leading dimension 36; tile column J starts at
// 576 J (J + 1) (all earlier tile columns are full); the last tile column
// is only as wide as needed.  Lower parts of diagonal tiles are zero.
#pragma once

#include "common.cuh"

namespace tfk {

constexpr int kTLD = 36;

__host__ __device__ __forceinline__ int tpu_w(int J, int K) { return min(32, K - 32 * J); }
__host__ __device__ __forceinline__ int64_t tpu_coff(int J) { return 576LL * J * (J + 1); }
__host__ __device__ __forceinline__ int64_t tpu_size(int K) {
  const int nb = (K + 31) / 32;
  return tpu_coff(nb - 1) + (int64_t)kTLD * nb * tpu_w(nb - 1, K);
}
__host__ __device__ __forceinline__ int64_t tpu_tile(int K, int I, int J) {
  return tpu_coff(J) + (int64_t)I * tpu_w(J, K) * kTLD;
}
// element (r, c); valid for r <= c or r, c in the same diagonal tile
__host__ __device__ __forceinline__ int64_t tpu_idx(int K, int r, int c) {
  const int J = c >> 5, I = r >> 5;
  return tpu_tile(K, I, J) + (int64_t)(c & 31) * kTLD + (r & 31);
}
__device__ __forceinline__ double tpu_get(const double* M, int K, int r, int c) {
  return (r <= c) ? M[tpu_idx(K, r, c)] : 0.0;
}

// Row loader of the reversed (target-first) weighted system of RH lag p on the
// p_bar-wide rows: a_t[a] = w_t y[base + i_t - a], a = 0..p (base = p_bar;
// column 0 is the target y[p_bar + i], column a >= 1 is lag a; sketch.cpp:61-79
// with width p).  Lag p - 1 is the leading p columns of lag p.
struct RevRows {
  const double* y;
  const int64_t* idx;
  const double* wt;
  int64_t base;
  __device__ __forceinline__ double operator()(int64_t t, int col) const {
    return wt[t] * y[base + idx[t] - col];
  }
};

// Row loader of the forward-ordered, weighted sampled system.
struct FwdRows {
  const double* y;
  const int64_t* idx;
  const double* wt;
  int64_t off;  // LSAR window system: 0; RH lag p on the full system: p_bar - p
  __device__ __forceinline__ double operator()(int64_t t, int col) const {
    return wt[t] * y[off + idx[t] + col];
  }
};

// ---------------------------------------------------------------------------
// Solve-state flags (per context): [0] shifted (pass A broke down),
// [1] failed, [2] need pass B, [3] unused.
struct SolveFlags {
  int* f;
};

// phi from S (TPU, K = p + 1) -> natural-order phi, packed coefficients, tau.
// S is the last of (SA, SB, SC) that was formed: SC if shifted, else SB if
// pass B ran, else SA.
struct PhiSArgs {
  int K;
  const double* SA;
  const double* SB;
  const double* SC;
  const int* flags;
  double* phi;        // natural order, length p
  double* coefs;      // nullable
  int64_t coef_off;
  double* taus;       // nullable
  int* method;        // nullable
  int lag;            // 1-based
  double* S_final;    // the final S (TPU): written by the last pass, read here and by the next lag
  int rev;            // column order: 0 forward (target last), 1 reversed (target first)
  double* rest_out;   // rev: 1 / ||S[0, :]||^2 (squared sampled residual norm) for the next lag
};

__global__ void k_phi_S(PhiSArgs a) {
  const int K = a.K, p = K - 1;
  const int* fl = a.flags;
  if (fl[1]) {
    for (int q = threadIdx.x; q < p; q += blockDim.x) a.phi[q] = __longlong_as_double(0x7ff8000000000000ll);
    return;
  }
  const double* S = a.S_final;  // the last S formed (every pass writes its S there too)
  if (a.rev) {
    // target first: v = S s0 / ||s0||^2 (s0 = row 0 of S) minimises ||A v|| with
    // v[0] = 1, so phi[j] = -v[1 + j] (natural order: column 1 + j is lag j + 1)
    __shared__ double red[32];
    double part = 0.0;
    for (int l = threadIdx.x; l < K; l += blockDim.x) {
      const double s0 = S[tpu_idx(K, 0, l)];
      part = fma(s0, s0, part);
    }
    part = warp_sum(part);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = part;
    __syncthreads();
    if (threadIdx.x < 32) {
      double x = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
      x = warp_sum(x);
      if (threadIdx.x == 0) red[0] = x;
    }
    __syncthreads();
    const double nrm2 = red[0];
    for (int q = threadIdx.x; q < p; q += blockDim.x) {
      const int j = q + 1;
      double acc = 0.0;
      for (int l = j; l < K; ++l) acc = fma(S[tpu_idx(K, j, l)], S[tpu_idx(K, 0, l)], acc);
      const double v = -acc / nrm2;
      a.phi[q] = v;
      if (a.coefs) a.coefs[a.coef_off + q] = v;
      if (a.taus && q == p - 1) a.taus[a.lag - 1] = v;
    }
    if (threadIdx.x == 0) {
      if (a.rest_out) a.rest_out[0] = 1.0 / nrm2;
      if (a.method) a.method[a.lag - 1] = fl[0] ? 3 : (fl[2] ? 2 : 1);
    }
    return;
  }
  const double spp = S[tpu_idx(K, p, p)];
  for (int q = threadIdx.x; q < p; q += blockDim.x) {
    const double v = -S[tpu_idx(K, p - 1 - q, p)] / spp;  // phi[q] = phi_fwd[p-1-q]
    a.phi[q] = v;
    if (a.coefs) a.coefs[a.coef_off + q] = v;
  }
  if (threadIdx.x == 0) {
    if (a.taus) a.taus[a.lag - 1] = -S[tpu_idx(K, 0, p)] / spp;
    if (a.method) a.method[a.lag - 1] = fl[0] ? 3 : (fl[2] ? 2 : 1);  // CholeskyQR passes used
  }
}

// T_{p} (TPU, K = p + 1) from S_{p-1} (TPU, K - 1), phi_{p-1} (natural
// order, length p - 1) and R_{p-1} = ||r_{p-1}||^2 (scal[0]).
__global__ void k_precond(const double* __restrict__ Sprev, const double* __restrict__ phi_prev,
                          const double* __restrict__ scal, double* __restrict__ T, int K) {
  const int p = K - 1;
  const double s = sqrt(fmax(scal[0], 1e-300));
  const double inv_s = 1.0 / s;
  const int64_t n = tpu_size(K);
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    // decode e -> (r, c)
    int J = 0;
    while (J + 1 < (K + 31) / 32 && tpu_coff(J + 1) <= e) ++J;
    const int64_t inJ = e - tpu_coff(J);
    const int wJ = tpu_w(J, K);
    const int I = (int)(inJ / ((int64_t)wJ * kTLD));
    const int64_t inT = inJ - (int64_t)I * wJ * kTLD;
    const int cc = (int)(inT / kTLD), rr = (int)(inT - (int64_t)cc * kTLD);
    double v = 0.0;
    if (rr < 32) {
      const int r = 32 * I + rr, c = 32 * J + cc;
      if (r <= c && r < K) {
        if (c < p) {
          v = Sprev[tpu_idx(K - 1, r, c)];
        } else if (r == p) {
          v = inv_s;
        } else {
          // target column: u[r] = -phi_fwd_prev[r - 1] / s, phi_fwd_prev[a] = phi_prev[p-2-a]
          v = r == 0 ? 0.0 : -phi_prev[p - 1 - r] * inv_s;
        }
      }
    }
    T[e] = v;
  }
}

// Identity preconditioner (first lag of a chain / standalone solves).
__global__ void k_tpu_identity(double* __restrict__ T, int K) {
  const int64_t n = tpu_size(K);
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    int J = 0;
    while (J + 1 < (K + 31) / 32 && tpu_coff(J + 1) <= e) ++J;
    const int64_t inJ = e - tpu_coff(J);
    const int wJ = tpu_w(J, K);
    const int I = (int)(inJ / ((int64_t)wJ * kTLD));
    const int64_t inT = inJ - (int64_t)I * wJ * kTLD;
    const int cc = (int)(inT / kTLD), rr = (int)(inT - (int64_t)cc * kTLD);
    T[e] = (I == J && rr == cc) ? 1.0 : 0.0;
  }
}

// p = 1 (K = 2): phi = a^T b / a^T a (exact when b is a power-of-two multiple
// of a, test_lsar.cpp:160-169) and S_1 = R^-1 of the 2x2 Gram (forward order:
// column 0 = y[i], column 1 = target y[i+1]).
__global__ void k_solve_k2(const double* G, PhiSArgs a) {
  const double g00 = G[tpu_idx(2, 0, 0)], g01 = G[tpu_idx(2, 0, 1)], g11 = G[tpu_idx(2, 1, 1)];
  const double phi = a.rev ? g01 / g11 : g01 / g00;  // rev: column 0 is the target
  a.phi[0] = phi;
  if (a.coefs) a.coefs[a.coef_off] = phi;
  if (a.taus) a.taus[a.lag - 1] = phi;
  if (a.method) a.method[a.lag - 1] = 0;
  if (a.S_final) {
    const double r00 = sqrt(g00), r01 = g01 / r00;
    double piv = g11 - r01 * r01;
    const double floor = 4.930380657631324e-32 * (g00 + g11);
    if (!(piv > floor)) piv = floor;
    const double r11 = sqrt(piv);
    a.S_final[tpu_idx(2, 0, 0)] = 1.0 / r00;
    a.S_final[tpu_idx(2, 0, 1)] = -r01 / (r00 * r11);
    a.S_final[tpu_idx(2, 1, 1)] = 1.0 / r11;
    a.S_final[tpu_idx(2, 1, 0)] = 0.0;
    if (a.rev && a.rest_out) {
      const double s00 = 1.0 / r00, s01 = -r01 / (r00 * r11);
      a.rest_out[0] = 1.0 / (s00 * s00 + s01 * s01);
    } else if (a.rest_out) {
      a.rest_out[0] = piv;  // forward order: ||r||^2 = g11 - g01^2 / g00
    }
  }
}

}  // namespace tfk
