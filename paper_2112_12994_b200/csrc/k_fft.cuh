// k_fft.cuh -- the LSAR pass with the FIR done as an overlap-save FFT
// convolution (fp64), for the long lags where the direct p-tap FIR is
// fp64-bound.
//
// The pass computes, per lag q over the w window rows (lsar.cpp:17-25,
// toeplitz.cpp:87-98):
//   r_q(i) = sum_{k=0..q} h_q[k] y[q + i - k],  h_q = [-1, phi_q[0..q-1]]
//   s_q(i) = s_{q-1}(i) + r_{q-1}(i)^2 / R_{q-1}
// plus the 32-row chunk / 2048-row tile partial sums of s_q and r_q^2 -- the
// same outputs, layout and update formula as k_lsar_pass_pst (k_pass.cuh).
//
// Overlap-save with N = 4096-point blocks: the filter f_q[D - q + k] = h_q[k]
// (delay D - q, D = 1024) makes every output row of a block land at the same
// position m = u + D of the circular convolution of x_j[m] = y[j L + m]
// (L = 3072 rows per block, no wrap-around for q <= D).  Two consecutive
// blocks a, b ride in one complex transform (x_a + i x_b): the series spectra
// Zab = DFT(x_a + i x_b) are computed ONCE per sweep (k_fft_series_dd, 64 KB per
// 6144-row superblock = 10.7 B per row), and per lag the pass multiplies by
// H = DFT(f_q) / N (k_fft_taps_dd) and inverts:
//   IDFT(Zab H) = (x_a (*) f_q) + i (x_b (*) f_q)
// -- the real part holds block a's residuals, the imaginary part block b's.
// Per row and lag: 10.7 B spectrum + 16 B (s, r) read + 16 B (s, r) written,
// ~40 fp64 operations, independent of q (the direct FIR: 2q + 4 flop).
//
// FFT: radix-16 Stockham autosort (three stages, 256 threads x 16 points in
// registers, two shared-memory exchanges through a padded buffer -- one slot
// per 16 complex values keeps every 16-byte access pattern conflict free).
// Stage 1 takes its input x[t + 256 r] straight from registers and stage 3
// leaves X[t + 256 r] (natural order) in registers, so for fixed r a warp's
// outputs are 32 consecutive rows: coalesced state loads / stores and chunk
// sums by warp shuffles.  Twiddles from two 256-entry tables in shared
// memory (W_256^e and W_4096^e, long-double accurate on the host);
// W_4096^{t r} = W_256^{(t>>4) r} W_4096^{(t&15) r}.
//
// Rounding: a plain fp64 FFT spreads an absolute error ~eps ||x|| over every
// bin of the series spectrum and ~eps ||h|| over every bin of the filter
// spectrum; the inverse filter H is large exactly where the series spectrum
// is small, so those errors come out amplified (C2 at q = 200: 1.6e-9 of
// max|r|, vs 4.9e-10 for the direct FIR's own rounding).  Both spectra are
// therefore computed in double-double and rounded once to fp64 (per bin
// relative error eps): k_fft_series_dd (a double-double Stockham FFT, once
// per sweep) and k_fft_taps_dd (a double-double direct DFT of the q + 1 taps,
// per lag).  The per-lag product and inverse FFT stay fp64: their errors are
// relative to the (small) residual spectrum.  Measured (tools/fft_precision.py,
// long double model): C2 1.2e-10 of max|r| vs the exact residuals -- 4x below
// the direct FIR's 4.9e-10; C4-shaped 8.7e-7 vs the direct FIR's 6.7e-6.
#pragma once

#include "common.cuh"
#include "k_exact.cuh"
#include "k_pass.cuh"

namespace tfk {

constexpr int kFftN = 4096;
constexpr int kFftT = 256;                       // threads per CTA, 16 points each
constexpr int kFftD = 1024;                      // filter delay: q <= kFftD
constexpr int kFftL = kFftN - kFftD;             // 3072 rows per block
constexpr int kFftSB = 2 * kFftL;                // 6144 rows per superblock (blocks a, b)
constexpr int kFftTilesSB = kFftSB / kPassTile;  // 3 tiles
constexpr int kFftChunksSB = kFftSB / kChunk;    // 192 chunks
constexpr int kFftBufC = kFftN + kFftN / 16;     // padded complex slots
constexpr int kFftTw = 512;                      // twiddle table entries (W_256^e, W_4096^e; e < 256)

__host__ __device__ __forceinline__ int fpad(int e) { return e + (e >> 4); }

inline size_t fft_smem_bytes(int tw_entries = kFftTw) { return sizeof(double2) * (size_t)(kFftBufC + tw_entries); }

__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
// a * w (S = -1, forward) or a * conj(w) (S = +1, inverse); w = e^{-2 pi i e / n} from the tables
template <int S>
__device__ __forceinline__ double2 ctw(double2 a, double2 w) {
  if (S < 0) return cmul(a, w);
  return make_double2(fma(a.x, w.x, a.y * w.y), fma(a.y, w.x, -a.x * w.y));
}

// 4-point DFT (sign S): y_k = sum_n x_n e^{S 2 pi i n k / 4}
template <int S>
__device__ __forceinline__ void dft4(double2& x0, double2& x1, double2& x2, double2& x3) {
  const double2 a = cadd(x0, x2), b = csub(x0, x2), c = cadd(x1, x3), d = csub(x1, x3);
  x0 = cadd(a, c);
  x2 = csub(a, c);
  if (S < 0) {  // b -+ i d
    x1 = make_double2(b.x + d.y, b.y - d.x);
    x3 = make_double2(b.x - d.y, b.y + d.x);
  } else {
    x1 = make_double2(b.x - d.y, b.y + d.x);
    x3 = make_double2(b.x + d.y, b.y - d.x);
  }
}

// x * e^{S 2 pi i m / 16}, m = n2 k1 in {1, 2, 3, 4, 6, 9}
template <int S, int M>
__device__ __forceinline__ double2 w16(double2 x) {
  constexpr double C1 = 0.92387953251128675613, S1 = 0.38268343236508977173, R2 = 0.70710678118654752440;
  if (M == 4) return S < 0 ? make_double2(x.y, -x.x) : make_double2(-x.y, x.x);
  constexpr double c = M == 1 ? C1 : M == 2 ? R2 : M == 3 ? S1 : M == 6 ? -R2 : -C1;
  constexpr double s0 = M == 1 ? S1 : M == 2 ? R2 : M == 3 ? C1 : M == 6 ? R2 : -S1;
  constexpr double s = S < 0 ? -s0 : s0;
  return make_double2(fma(x.x, c, -x.y * s), fma(x.x, s, x.y * c));
}

// 16-point DFT in registers (4 x 4); the result replaces v in natural order
template <int S>
__device__ __forceinline__ void fft16(double2 (&v)[16]) {
#pragma unroll
  for (int n2 = 0; n2 < 4; ++n2) dft4<S>(v[n2], v[4 + n2], v[8 + n2], v[12 + n2]);
  // v[4 k1 + n2] *= W16^{n2 k1}
  v[5] = w16<S, 1>(v[5]);
  v[6] = w16<S, 2>(v[6]);
  v[7] = w16<S, 3>(v[7]);
  v[9] = w16<S, 2>(v[9]);
  v[10] = w16<S, 4>(v[10]);
  v[11] = w16<S, 6>(v[11]);
  v[13] = w16<S, 3>(v[13]);
  v[14] = w16<S, 6>(v[14]);
  v[15] = w16<S, 9>(v[15]);
#pragma unroll
  for (int k1 = 0; k1 < 4; ++k1) dft4<S>(v[4 * k1], v[4 * k1 + 1], v[4 * k1 + 2], v[4 * k1 + 3]);
  // X[k1 + 4 k2] sits at v[4 k1 + k2]: transpose (register renaming)
  double2 o[16];
#pragma unroll
  for (int r = 0; r < 16; ++r) o[r] = v[4 * (r & 3) + (r >> 2)];
#pragma unroll
  for (int r = 0; r < 16; ++r) v[r] = o[r];
}

// 4096-point DFT (sign S, unnormalised) of x[t + 256 r] = v[r] (thread t of
// 256); on return v[r] = X[t + 256 r].  buf: kFftBufC padded slots; tw: the
// two twiddle tables in shared memory.  Begins with a barrier (buf may still be
// read by the previous call) and ends without one.
// v[r] *= w1^r (S = -1) or conj(w1)^r (S = +1), r = 1..15, the powers formed
// in registers from the one table entry w1: 14 complex products at depth <= 5
// (w2 = w1^2, w3 = w2 w1, w4 = w2^2, w8 = w4^2, w12 = w8 w4 and the bases times
// w1..w3) in place of 15 (stage 2) / 30 (stage 3) 16-byte shared-memory loads
// per thread -- those loads were half of the transform's shared-memory
// wavefronts (index (t & 15) r: stride-r bank conflicts), on the L1 pipe that
// bounds the pass.  The powers carry <= ~8 eps of relative error, like the
// transform's own rounding: relative to the residual spectrum (see Rounding).
template <int S>
__device__ __forceinline__ void tw_powers(double2 (&v)[16], double2 w1) {
  const double2 w2 = cmul(w1, w1), w3 = cmul(w2, w1), w4 = cmul(w2, w2);
  v[1] = ctw<S>(v[1], w1);
  v[2] = ctw<S>(v[2], w2);
  v[3] = ctw<S>(v[3], w3);
  v[4] = ctw<S>(v[4], w4);
  double2 b = w4;
#pragma unroll
  for (int g = 1; g < 4; ++g) {
    v[4 * g + 1] = ctw<S>(v[4 * g + 1], cmul(b, w1));
    v[4 * g + 2] = ctw<S>(v[4 * g + 2], cmul(b, w2));
    v[4 * g + 3] = ctw<S>(v[4 * g + 3], cmul(b, w3));
    if (g < 3) {
      b = cmul(b, w4);
      v[4 * g + 4] = ctw<S>(v[4 * g + 4], b);
    }
  }
}

// TW: 0 twiddles from the two tables (W_256^{(t&15) r}; W_256^{(t>>4) r} W_4096^{(t&15) r}),
// 1 powers of one table entry per stage (tw_powers)
// (the tables then need only W_256^e, e < 16, and W_4096^e, e < 256: fft_tw_entries)
template <int S, int TW = 0>
__device__ __forceinline__ void fft4096(double2 (&v)[16], double2* buf, const double2* tw) {
  const int t = threadIdx.x;
  const double2* tw256 = tw;
  const double2* twlo = tw + (TW == 1 ? 16 : 256);
  // stage 1 (Ns = 1): no twiddles; out -> buf[16 t + r]
  fft16<S>(v);
  __syncthreads();
#pragma unroll
  for (int r = 0; r < 16; ++r) buf[fpad(16 * t + r)] = v[r];
  __syncthreads();
  // stage 2 (Ns = 16): twiddle W_256^{(t & 15) r}; out -> buf[(t >> 4) 256 + (t & 15) + 16 r]
#pragma unroll
  for (int r = 0; r < 16; ++r) v[r] = buf[fpad(t + 256 * r)];
  if (TW == 1) {
    tw_powers<S>(v, tw256[t & 15]);
  } else {
#pragma unroll
    for (int r = 1; r < 16; ++r) v[r] = ctw<S>(v[r], tw256[(t & 15) * r]);
  }
  fft16<S>(v);
  __syncthreads();
  const int d2 = (t >> 4) * 256 + (t & 15);
#pragma unroll
  for (int r = 0; r < 16; ++r) buf[fpad(d2 + 16 * r)] = v[r];
  __syncthreads();
  // stage 3 (Ns = 256): twiddle W_4096^{t r} = W_256^{(t >> 4) r} W_4096^{(t & 15) r}; natural order out
#pragma unroll
  for (int r = 0; r < 16; ++r) v[r] = buf[fpad(t + 256 * r)];
  if (TW == 1) {
    tw_powers<S>(v, twlo[t]);  // W_4096^t
  } else {
#pragma unroll
    for (int r = 1; r < 16; ++r) v[r] = ctw<S>(v[r], cmul(tw256[(t >> 4) * r], twlo[(t & 15) * r]));
  }
  fft16<S>(v);
}

// shared-memory twiddle entries: TW 0 both 256-entry tables, TW 1 W_256^e (e < 16) + W_4096^e (e < 256)
template <int TW>
__host__ __device__ constexpr int fft_tw_entries() { return TW == 1 ? 16 + 256 : kFftTw; }
template <int TW = 0>
__device__ __forceinline__ void fft_load_tw(double2* tw_s, const double2* tw_g) {
  if (TW == 1) {
    for (int e = threadIdx.x; e < 16 + 256; e += blockDim.x) tw_s[e] = tw_g[e < 16 ? e : 256 + (e - 16)];
  } else {
    for (int e = threadIdx.x; e < kFftTw; e += blockDim.x) tw_s[e] = tw_g[e];
  }
}

// ---------------------------------------------------------------------------
// ---------------------------------------------------------------------------
// Double-double spectra (both rounded once to fp64 at the end).
struct CD {
  DD x, y;
};
__device__ __forceinline__ CD cd_add(const CD& a, const CD& b) { return {dd_add(a.x, b.x), dd_add(a.y, b.y)}; }
__device__ __forceinline__ CD cd_sub(const CD& a, const CD& b) {
  return {dd_add(a.x, dd_neg(b.x)), dd_add(a.y, dd_neg(b.y))};
}
__device__ __forceinline__ CD cd_mul(const CD& a, const CD& b) {
  return {dd_add(dd_mul(a.x, b.x), dd_neg(dd_mul(a.y, b.y))), dd_add(dd_mul(a.x, b.y), dd_mul(a.y, b.x))};
}
// forward 4-point DFT (e^{-2 pi i n k / 4}); multiplications by -i are exact
__device__ __forceinline__ void dft4_dd(CD& x0, CD& x1, CD& x2, CD& x3) {
  const CD a = cd_add(x0, x2), b = cd_sub(x0, x2), c = cd_add(x1, x3), d = cd_sub(x1, x3);
  x0 = cd_add(a, c);
  x2 = cd_sub(a, c);
  x1 = {dd_add(b.x, d.y), dd_add(b.y, dd_neg(d.x))};  // b - i d
  x3 = {dd_add(b.x, dd_neg(d.y)), dd_add(b.y, d.x)};  // b + i d
}
// twiddle tables in shared memory: [0, 256) W_256^e, [256, 512) W_4096^e (hi; lo in a parallel array)
struct TwDD {
  const double2* h;
  const double2* l;
  __device__ __forceinline__ CD operator[](int e) const {
    const double2 a = h[e], b = l[e];
    return {DD{a.x, b.x}, DD{a.y, b.y}};
  }
};
__device__ __forceinline__ void fft16_dd(CD (&v)[16], const TwDD& tw) {
#pragma unroll
  for (int n2 = 0; n2 < 4; ++n2) dft4_dd(v[n2], v[4 + n2], v[8 + n2], v[12 + n2]);
  // v[4 k1 + n2] *= W16^{n2 k1} = W_256^{16 n2 k1}; n2 k1 = 4: -i (exact)
  v[5] = cd_mul(v[5], tw[16]);
  v[6] = cd_mul(v[6], tw[32]);
  v[7] = cd_mul(v[7], tw[48]);
  v[9] = cd_mul(v[9], tw[32]);
  v[10] = CD{v[10].y, dd_neg(v[10].x)};
  v[11] = cd_mul(v[11], tw[96]);
  v[13] = cd_mul(v[13], tw[48]);
  v[14] = cd_mul(v[14], tw[96]);
  v[15] = cd_mul(v[15], tw[144]);
#pragma unroll
  for (int k1 = 0; k1 < 4; ++k1) dft4_dd(v[4 * k1], v[4 * k1 + 1], v[4 * k1 + 2], v[4 * k1 + 3]);
  CD o[16];
#pragma unroll
  for (int r = 0; r < 16; ++r) o[r] = v[4 * (r & 3) + (r >> 2)];
#pragma unroll
  for (int r = 0; r < 16; ++r) v[r] = o[r];
}
__device__ __forceinline__ void cd_st(double2* bh, double2* bl, int i, const CD& a) {
  bh[i] = make_double2(a.x.h, a.y.h);
  bl[i] = make_double2(a.x.l, a.y.l);
}
__device__ __forceinline__ CD cd_ld(const double2* bh, const double2* bl, int i) {
  const double2 a = bh[i], b = bl[i];
  return {DD{a.x, b.x}, DD{a.y, b.y}};
}
// forward 4096-point DFT in double-double, same data flow as fft4096<-1>
__device__ __forceinline__ void fft4096_dd(CD (&v)[16], double2* bh, double2* bl, const TwDD& tw) {
  const int t = threadIdx.x;
  fft16_dd(v, tw);
  __syncthreads();
#pragma unroll
  for (int r = 0; r < 16; ++r) cd_st(bh, bl, fpad(16 * t + r), v[r]);
  __syncthreads();
#pragma unroll
  for (int r = 0; r < 16; ++r) v[r] = cd_ld(bh, bl, fpad(t + 256 * r));
#pragma unroll
  for (int r = 1; r < 16; ++r) v[r] = cd_mul(v[r], tw[(t & 15) * r]);
  fft16_dd(v, tw);
  __syncthreads();
  const int d2 = (t >> 4) * 256 + (t & 15);
#pragma unroll
  for (int r = 0; r < 16; ++r) cd_st(bh, bl, fpad(d2 + 16 * r), v[r]);
  __syncthreads();
#pragma unroll
  for (int r = 0; r < 16; ++r) v[r] = cd_ld(bh, bl, fpad(t + 256 * r));
#pragma unroll
  for (int r = 1; r < 16; ++r) v[r] = cd_mul(v[r], cd_mul(tw[(t >> 4) * r], tw[256 + (t & 15) * r]));
  fft16_dd(v, tw);
}

inline size_t fft_dd_smem_bytes() { return 2 * sizeof(double2) * (size_t)(kFftBufC + kFftTw); }

// Series spectra, once per sweep: Zab[sb][k] = DFT(x_a + i x_b)[k] with
// x_a[m] = y[6144 sb + m], x_b[m] = y[6144 sb + 3072 + m] (0 past n), in
// double-double, rounded to fp64.  twh / twl: W_4096^e, e < 4096 (hi, lo).
__global__ void __launch_bounds__(kFftT, 1) k_fft_series_dd(const double* __restrict__ y, int64_t n, int64_t nsb,
                                                            double2* __restrict__ Z, const double2* __restrict__ twh,
                                                            const double2* __restrict__ twl) {
  extern __shared__ double2 fsm[];
  double2* bh = fsm;
  double2* bl = fsm + kFftBufC;
  double2* th = fsm + 2 * kFftBufC;
  double2* tl = th + kFftTw;
  for (int e = threadIdx.x; e < 256; e += blockDim.x) {
    th[e] = twh[16 * e];  // W_256^e
    tl[e] = twl[16 * e];
    th[256 + e] = twh[e];  // W_4096^e
    tl[256 + e] = twl[e];
  }
  __syncthreads();
  const TwDD tw{th, tl};
  const int t = threadIdx.x;
  for (int64_t sb = blockIdx.x; sb < nsb; sb += gridDim.x) {
    const int64_t ia = sb * kFftSB + t, ib = ia + kFftL;
    CD v[16];
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      const int64_t a = ia + 256 * r, b = ib + 256 * r;
      v[r] = CD{DD{a < n ? __ldg(y + a) : 0.0, 0.0}, DD{b < n ? __ldg(y + b) : 0.0, 0.0}};
    }
    fft4096_dd(v, bh, bl, tw);
    double2* Zs = Z + sb * kFftN + t;
#pragma unroll
    for (int r = 0; r < 16; ++r) __stcs(Zs + 256 * r, make_double2(v[r].x.h, v[r].y.h));
  }
}

// Per lag: H[k] = DFT(f_q)[k] / N, f_q[D - q + j] = h_q[j] (h_q[0] = -1,
// h_q[j] = phi[j - 1]) as a direct DFT of the q + 1 taps in double-double
// (the products h_j W are exact-ish: 2 fp64 x double-double), rounded to
// fp64.  256 threads = 32 bins x 8 tap slices; slices summed by a fixed
// butterfly; grid 4096 / 32.
constexpr int kTapSplit = 8;
__global__ void __launch_bounds__(256) k_fft_taps_dd(const double* __restrict__ phi, int q, double2* __restrict__ H,
                                                     const double2* __restrict__ twh,
                                                     const double2* __restrict__ twl) {
  const int t = threadIdx.x, sl = t & (kTapSplit - 1);
  const int k = blockIdx.x * (256 / kTapSplit) + (t / kTapSplit);
  const int per = (q + kTapSplit) / kTapSplit;  // ceil((q + 1) / 8)
  const int j0 = sl * per, j1 = min(q + 1, j0 + per);
  DD re{0.0, 0.0}, im{0.0, 0.0};
  for (int j = j0; j < j1; ++j) {
    const double hj = j == 0 ? -1.0 : __ldg(phi + j - 1);
    const int e = ((kFftD - q + j) * k) & (kFftN - 1);
    const double2 wh = __ldg(twh + e), wl = __ldg(twl + e);
    re = dd_add(re, dd_mul(DD{hj, 0.0}, DD{wh.x, wl.x}));
    im = dd_add(im, dd_mul(DD{hj, 0.0}, DD{wh.y, wl.y}));
  }
#pragma unroll
  for (int m = 1; m < kTapSplit; m <<= 1) {
    const DD ro{__shfl_xor_sync(0xffffffffu, re.h, m), __shfl_xor_sync(0xffffffffu, re.l, m)};
    const DD io{__shfl_xor_sync(0xffffffffu, im.h, m), __shfl_xor_sync(0xffffffffu, im.l, m)};
    // lower slice first: the same operand order in every lane of the pair
    re = (sl & m) ? dd_add(ro, re) : dd_add(re, ro);
    im = (sl & m) ? dd_add(io, im) : dd_add(im, io);
  }
  constexpr double inv = 1.0 / kFftN;  // exact (power of two)
  if (sl == 0) H[k] = make_double2(re.h * inv, im.h * inv);
}

// Deterministic warp reduction of 12 values per lane: on return x[0] of lane
// (b4 b3 b2 b1 b0) holds the sum over the warp of value 6 b4 + 3 b3 + 2 b2 + b1
// (none when 2 b2 + b1 == 3; both b0 lanes hold it).  13 shuffles instead of
// 12 x 5; every value is summed over the lane pairs xor 16, 8, 4, 2, 1 in that
// order (a + b on both lanes of a pair: the same bits everywhere).
__device__ __forceinline__ void warp_reduce12(double (&x)[12], int lane) {
  const bool b4 = lane & 16, b3 = lane & 8, b2 = lane & 4, b1 = lane & 2;
#pragma unroll
  for (int i = 0; i < 6; ++i) {
    const double snd = b4 ? x[i] : x[i + 6];
    const double rcv = __shfl_xor_sync(0xffffffffu, snd, 16);
    x[i] = (b4 ? x[i + 6] : x[i]) + rcv;
  }
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const double snd = b3 ? x[i] : x[i + 3];
    const double rcv = __shfl_xor_sync(0xffffffffu, snd, 8);
    x[i] = (b3 ? x[i + 3] : x[i]) + rcv;
  }
  x[3] = 0.0;
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const double snd = b2 ? x[i] : x[i + 2];
    const double rcv = __shfl_xor_sync(0xffffffffu, snd, 4);
    x[i] = (b2 ? x[i + 2] : x[i]) + rcv;
  }
  {
    const double snd = b1 ? x[0] : x[1];
    const double rcv = __shfl_xor_sync(0xffffffffu, snd, 2);
    x[0] = (b1 ? x[1] : x[0]) + rcv;
  }
  x[0] += __shfl_xor_sync(0xffffffffu, x[0], 1);
}

// Deferred score folding (kFftSlots residual arrays): the fold of r_j^2 / R_j
// into s is per row a read-modify-write of s (16 B/row), so it is done for one
// group of superblocks per lag -- group g = (sb + sb / grid) mod K (each CTA of
// the persistent grid folds every K-th superblock it visits) folds at the lags
// q0 + g + m K and then adds its K pending residuals r_{q-K} .. r_{q-1} in lag
// order (the same fma sequence per row as one fold per lag).  The
// other K - 1 groups only read the spectrum and write r_q (18.7 B/row), their
// 32-row chunk sums of s advanced by the chunk recurrence A_q = A_{q-1} +
// B_{q-1} / R_{q-1}.  Residual r_j lives in slot (j - q0 + 1) mod (K + 1) until
// every group has folded it (K + 1 slots: r_q never lands on a pending residual,
// so the pass writes r_q first -- its transform registers are then free -- and
// folds afterwards with every pending load of 12 rows in flight at once); a
// draw at a row computes the exact s_{q+1}(row) from s and the row group's
// pending residuals (PendState).  K = 1: one fold per lag for every superblock
// (s_q and r_q in place: r_{q-1} is loaded before r_q is stored).
constexpr int kFftSlots = 4;

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((uint32_t)__cvta_generic_to_shared(smem)), "l"(gmem)
               : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

struct FftPassArgs {
  const double2* Z;  // [nsb][4096] series spectra (k_fft_series_dd)
  const double2* H;  // [4096] filter spectrum of this lag / N (k_fft_taps_dd)
  const double2* tw;
  int64_t w;
  double* s;  // the folded scores of the folding group (in place)
  int K;      // superblock groups (1: every superblock folds every lag)
  int fold;   // the group folding at this lag
  int npend;  // its pending residuals (oldest first), 1..K
  const double* pend[kFftSlots];
  const double* Rp;  // R of the pending lags [npend]; Rp[npend - 1] = R_{q-1}
  double* rout;      // r_q (K = 1: aliases pend[0], which is then loaded before the store)
  double* chunkA;
  double* chunkB;
  double* tileA;
  double* tileB;
  int ggrid;  // the grid the superblock groups are defined on: group(sb) = (sb + sb / ggrid) mod K
  int split;  // 1: the scores (phase 2 below) are k_fft_fold's, on another stream; the pass writes r_q, B only
};

__device__ __forceinline__ bool fft_folds(const FftPassArgs& a, int64_t sb) {
  // (32-bit arithmetic: the superblock index is far below 2^32)
  return a.K == 1 || (int)(((uint32_t)sb + (uint32_t)sb / (uint32_t)a.ggrid) % (uint32_t)a.K) == a.fold;
}

// Phase 2 of a superblock (K > 1), by the 256 threads of a CTA: the chunk sums
// of s_q into csA / chunkA.  Folding superblock: s += the pending r_j^2 / R_j
// in lag order; per block half every load of s and two pending residuals (36
// per thread) is in flight at once.  Otherwise the chunk recurrence A_q =
// A_{q-1} + B_{q-1} / R_{q-1} on (oA, oB) = the chunk sums of lag q - 1.
// Shared by the fused pass and k_fft_fold: the same operations, the same bits.
__device__ __forceinline__ void fft_scores_phase(const FftPassArgs& a, int64_t sb, bool fold, double* csA,
                                                 const double* invRp, double oA, double oB) {
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int64_t w = a.w;
  const int64_t base = sb * kFftSB + t;
  double* __restrict__ sp = a.s;
  // reduced value i = 6 b4 + 3 b3 + 2 b2 + b1 of warp_reduce12 -> its chunk; one writer lane per value
  const int vi = 6 * ((lane >> 4) & 1) + 3 * ((lane >> 3) & 1) + ((lane >> 1) & 3);
  const bool writer = (lane & 1) == 0 && ((lane >> 1) & 3) != 3;
  if (fold) {
#pragma unroll 1
    for (int h = 0; h < 2; ++h) {
      double so[12], ra[12], rb[12];
      const bool two = a.npend > 1;
#pragma unroll
      for (int i = 0; i < 12; ++i) {
        const int64_t row = base + h * kFftL + 256 * i;
        const bool ok = row < w;
        so[i] = ok ? __ldcs(sp + row) : 0.0;
        ra[i] = ok ? __ldcs(a.pend[0] + row) : 0.0;
        rb[i] = ok && two ? __ldcs(a.pend[1] + row) : 0.0;
      }
#pragma unroll
      for (int i = 0; i < 12; ++i) so[i] = fma(ra[i] * ra[i], invRp[0], so[i]);
      if (two) {
#pragma unroll
        for (int i = 0; i < 12; ++i) so[i] = fma(rb[i] * rb[i], invRp[1], so[i]);
      }
      if (a.npend > 2) {
        const bool four = a.npend > 3;
#pragma unroll
        for (int i = 0; i < 12; ++i) {
          const int64_t row = base + h * kFftL + 256 * i;
          const bool ok = row < w;
          ra[i] = ok ? __ldcs(a.pend[2] + row) : 0.0;
          rb[i] = ok && four ? __ldcs(a.pend[3] + row) : 0.0;
        }
#pragma unroll
        for (int i = 0; i < 12; ++i) so[i] = fma(ra[i] * ra[i], invRp[2], so[i]);
        if (four) {
#pragma unroll
          for (int i = 0; i < 12; ++i) so[i] = fma(rb[i] * rb[i], invRp[3], so[i]);
        }
      }
#pragma unroll
      for (int i = 0; i < 12; ++i) {
        const int64_t row = base + h * kFftL + 256 * i;
        if (row < w) __stcs(sp + row, so[i]);
        else so[i] = 0.0;
      }
      warp_reduce12(so, lane);
      const int cl = 96 * h + 8 * vi + warp;
      const int64_t cg = sb * kFftChunksSB + cl;
      if (writer) {
        csA[cl] = so[0];
        if (cg * kChunk < w) a.chunkA[cg] = so[0];
      }
    }
  } else if (t < kFftChunksSB) {
    const int64_t cg = sb * kFftChunksSB + t;
    const bool live = cg * kChunk < w;
    const double nA = live ? fma(oB, invRp[a.npend - 1], oA) : 0.0;
    csA[t] = nA;
    if (live) a.chunkA[cg] = nA;
  }
}

// 2048-row tile sums of a superblock from its 192 chunk sums (warps 0..2, after a barrier)
__device__ __forceinline__ void fft_tile_sums(const double* cs, double* tile, int64_t sb, int64_t w) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (warp < kFftTilesSB) {
    const int64_t tg = sb * kFftTilesSB + warp;
    const double T = warp_sum(cs[64 * warp + lane] + cs[64 * warp + 32 + lane]);
    if (lane == 0 && tg * kPassTile < w) tile[tg] = T;
  }
}

// Persistent CTAs (2 per SM) over 6144-row superblocks.  PF (prefetch):
// 0 none, 1 the next superblock's spectrum + state to L2, 2 this superblock's
// state to L2 at the start of its iteration, 3 = 2 + the next superblock's
// spectrum to L2, 4 = 3 + the spectrum through shared memory by TMA (the
// default; profiles/r02_fft_prefetch.txt)
template <int PF, int TW = 0>
__global__ void __launch_bounds__(kFftT, 2) k_lsar_pass_fft(FftPassArgs a) {
  extern __shared__ double2 fsm[];
  __shared__ double coA[kFftChunksSB], coB[kFftChunksSB];  // non-folding superblock: chunk sums of lag q - 1
  double2* buf = fsm;
  double2* tw = fsm + kFftBufC;
  // this superblock's chunk sums live in the transform buffer's padding tail (slots 4096 ..: free
  // from the last transform stage's reads to the next superblock's first exchange; the next
  // spectrum's bulk copy fills slots [0, 4096) only).  Shared memory per CTA stays under 81 KB, so
  // two CTAs fit the 164 KB carve-out and the L1 beside it (~92 KB) keeps the 64 KB of H resident.
  double* csA = reinterpret_cast<double*>(buf + kFftN);
  double* csB = csA + kFftChunksSB;
  static_assert(2 * kFftChunksSB * sizeof(double) <= (kFftBufC - kFftN) * sizeof(double2), "chunk sums fit the padding");
  fft_load_tw<TW>(tw, a.tw);
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int64_t w = a.w;
  const int64_t nsb = (w + kFftSB - 1) / kFftSB;
  __shared__ double invRp[kFftSlots];  // 1 / R of the pending lags (shared: no registers held)
  if (t < kFftSlots) invRp[t] = t < a.npend ? 1.0 / a.Rp[t] : 0.0;
  // L2 prefetch (cp.async.bulk.prefetch) of a superblock's spectrum and state:
  // this CTA's first superblock's state now, the next one's inputs while the
  // current one computes -- the state loads after the FFT then hit L2
  auto prefetch = [&](int64_t p, bool spectrum) {
    if (p >= nsb) return;
    const int64_t r0 = p * kFftSB;
    const uint32_t bytes = (uint32_t)(min((int64_t)kFftSB, w - r0) * 8) & ~15u;
    if (spectrum) bulk_prefetch_l2(a.Z + p * kFftN, kFftN * sizeof(double2));
    if (bytes && !a.split && fft_folds(a, p)) {
      bulk_prefetch_l2(a.s + r0, bytes);
      for (int k = 0; k < a.npend; ++k) bulk_prefetch_l2(a.pend[k] + r0, bytes);
    }
  };
  // PF 4: the spectrum goes through shared memory -- a TMA bulk copy of the
  // next superblock's 64 KB spectrum into the (unpadded) transform buffer,
  // issued once this superblock's last transform stage has read the buffer,
  // so it lands during the state phase (the spectrum load was the top stall)
  __shared__ __align__(8) uint64_t zbar;
  constexpr uint32_t kZBytes = kFftN * sizeof(double2);
  if (PF == 4) {
    if (t == 0) mbar_init(&zbar, 1);
    __syncthreads();
    if (t == 0 && blockIdx.x < nsb) {
      mbar_expect_tx(&zbar, kZBytes);
      bulk_g2s(buf, a.Z + (int64_t)blockIdx.x * kFftN, kZBytes, &zbar);
    }
  }
  uint32_t zphase = 0;
  if (PF == 1 && t == 0) prefetch(blockIdx.x, false);
  for (int64_t sb = blockIdx.x; sb < nsb; sb += gridDim.x) {
    if (PF == 1 && t == 0) prefetch(sb + gridDim.x, true);
    if (PF >= 2 && t == 0) prefetch(sb, false);
    if (PF >= 3 && t == 0 && sb + gridDim.x < nsb)
      bulk_prefetch_l2(a.Z + (sb + gridDim.x) * kFftN, kFftN * sizeof(double2));
    // group of sb: (sb + sb / grid) mod K -- each CTA folds every K-th superblock it visits (balanced)
    const bool fold = fft_folds(a, sb);
    if (!a.split && !fold && t < kFftChunksSB) {  // the previous chunk sums, in flight during the transform
      const int64_t cg = sb * kFftChunksSB + t;
      if (cg * kChunk < w) {
        cp_async8(coA + t, a.chunkA + cg);
        cp_async8(coB + t, a.chunkB + cg);
      }
    }
    double2 v[16];
    if (PF == 4) {
      mbar_wait(&zbar, zphase);
      zphase ^= 1u;
#pragma unroll
      for (int r = 0; r < 16; ++r) v[r] = cmul(buf[t + 256 * r], __ldg(a.H + t + 256 * r));
    } else {
      const double2* Zs = a.Z + sb * kFftN + t;
#pragma unroll
      for (int r = 0; r < 16; ++r) v[r] = cmul(__ldcs(Zs + 256 * r), __ldg(a.H + t + 256 * r));
    }
    fft4096<1, TW>(v, buf, tw);
    cp_async_wait_all();
    __syncthreads();  // every thread's last-stage reads of buf are done; coA / coB landed
    if (PF == 4) {
      if (t == 0 && sb + gridDim.x < nsb) {
        fence_proxy_async_smem();
        mbar_expect_tx(&zbar, kZBytes);
        bulk_g2s(buf, a.Z + (sb + gridDim.x) * kFftN, kZBytes, &zbar);
      }
    }
    // rows: output m = t + 256 r (r >= 4) -> u = m - D; block a row base + u (real part), block b row
    // base + 3072 + u (imaginary part): for fixed r a warp holds the 32 rows of chunk 96 h + 8 (r - 4) + warp.
    const int64_t base = sb * kFftSB + t;
    double* __restrict__ sp = a.s;
    double* rp = a.rout;
    const bool alias = a.K == 1;  // rout == pend[0]: r_{q-1} comes in before r_q goes out
    // reduced value i = 6 b4 + 3 b3 + 2 b2 + b1 of warp_reduce12 -> its chunk; one writer lane per value
    const int vi = 6 * ((lane >> 4) & 1) + 3 * ((lane >> 3) & 1) + ((lane >> 1) & 3);
    const bool writer = (lane & 1) == 0 && ((lane >> 1) & 3) != 3;
    // (1) r_q out and the chunk sums of r_q^2 (K = 1: the fold of r_{q-1} first, 6 rows at a time)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      double x[12];
      if (alias) {
        double xs[12];
#pragma unroll
        for (int g = 0; g < 2; ++g) {
          double so[6], ro[6];
#pragma unroll
          for (int j = 0; j < 6; ++j) {
            const int64_t row = base + h * kFftL + 256 * (6 * g + j);
            so[j] = row < w ? __ldcs(sp + row) : 0.0;
            ro[j] = row < w ? __ldcs(a.pend[0] + row) : 0.0;
          }
#pragma unroll
          for (int j = 0; j < 6; ++j) {
            const int i = 6 * g + j;
            const int64_t row = base + h * kFftL + 256 * i;
            const double rq = h ? v[4 + i].y : v[4 + i].x;
            const double sn = fma(ro[j] * ro[j], invRp[0], so[j]);
            double rs = 0.0;
            if (row < w) {
              __stcs(sp + row, sn);
              __stcs(rp + row, rq);
              rs = rq;
            }
            xs[i] = row < w ? sn : 0.0;
            x[i] = rs * rs;
          }
        }
        warp_reduce12(xs, lane);
        const int cl = 96 * h + 8 * vi + warp;
        const int64_t cg = sb * kFftChunksSB + cl;
        if (writer) {
          csA[cl] = xs[0];
          if (cg * kChunk < w) a.chunkA[cg] = xs[0];
        }
      } else {
#pragma unroll
        for (int i = 0; i < 12; ++i) {
          const int64_t row = base + h * kFftL + 256 * i;
          const double rq = h ? v[4 + i].y : v[4 + i].x;
          double rs = 0.0;
          if (row < w) {
            __stcs(rp + row, rq);
            rs = rq;
          }
          x[i] = rs * rs;
        }
      }
      warp_reduce12(x, lane);
      const int cl = 96 * h + 8 * vi + warp;  // chunk of the superblock
      const int64_t cg = sb * kFftChunksSB + cl;
      if (writer) {
        csB[cl] = x[0];
        if (cg * kChunk < w) a.chunkB[cg] = x[0];
      }
    }
    // (2) the scores (K > 1; the transform's registers are dead) -- unless k_fft_fold computes them
    if (!alias && !a.split) fft_scores_phase(a, sb, fold, csA, invRp, t < kFftChunksSB ? coA[t] : 0.0, t < kFftChunksSB ? coB[t] : 0.0);
    __syncthreads();
    if (!a.split) fft_tile_sums(csA, a.tileA, sb, w);
    fft_tile_sums(csB, a.tileB, sb, w);
    // csA / csB are rewritten only after the next fft4096's barriers
  }
}

// The pass proper when the scores are k_fft_fold's (FftPassArgs::split, K > 1):
// transform -> r_q and the chunk / tile sums of r_q^2, nothing else.  With no
// fold in the kernel the transform registers are free as soon as r_q is stored,
// so the NEXT superblock's spectrum is loaded straight into them (16 coalesced
// 16-byte loads per thread, L2 hits: the spectrum was prefetched to L2 one
// superblock earlier) and is in flight over the reductions, the barrier, the
// tile sums and the loop edge -- no shared-memory staging of the spectrum (the
// bulk copy's 64 KB write and the 16 LDS.128 per thread were a quarter of the
// kernel's shared-memory wavefronts), no mbarrier.  Same arithmetic as
// k_lsar_pass_fft<4, 1>: the same bits.  MEASURED SLOWER than the TMA-staged
// spectrum at C4 (pass 3.66 vs 3.46 s per sweep, profiles/r02_fft_prefetch.txt):
// kept behind TF_FFT_RPF=1 as the record of the experiment, not the default.
__global__ void __launch_bounds__(kFftT, 2) k_lsar_pass_fft_r(FftPassArgs a) {
  extern __shared__ double2 fsm[];
  double2* buf = fsm;
  double2* tw = fsm + kFftBufC;
  double* csB = reinterpret_cast<double*>(buf + kFftN);  // the buffer's padding tail (see k_lsar_pass_fft)
  fft_load_tw<1>(tw, a.tw);
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int64_t w = a.w;
  const int64_t nsb = (w + kFftSB - 1) / kFftSB;
  const int vi = 6 * ((lane >> 4) & 1) + 3 * ((lane >> 3) & 1) + ((lane >> 1) & 3);
  const bool writer = (lane & 1) == 0 && ((lane >> 1) & 3) != 3;
  double2 v[16];
  if ((int64_t)blockIdx.x < nsb) {
    const double2* Zs = a.Z + (int64_t)blockIdx.x * kFftN + t;
#pragma unroll
    for (int r = 0; r < 16; ++r) v[r] = __ldcs(Zs + 256 * r);
    if (t == 0 && (int64_t)blockIdx.x + gridDim.x < nsb)
      bulk_prefetch_l2(a.Z + ((int64_t)blockIdx.x + gridDim.x) * kFftN, kFftN * sizeof(double2));
  }
  for (int64_t sb = blockIdx.x; sb < nsb; sb += gridDim.x) {
    if (t == 0 && sb + 2 * (int64_t)gridDim.x < nsb)
      bulk_prefetch_l2(a.Z + (sb + 2 * (int64_t)gridDim.x) * kFftN, kFftN * sizeof(double2));
#pragma unroll
    for (int r = 0; r < 16; ++r) v[r] = cmul(v[r], __ldg(a.H + t + 256 * r));
    fft4096<1, 1>(v, buf, tw);
    __syncthreads();  // every thread's last-stage reads of buf (its tail holds csB) are done
    const int64_t base = sb * kFftSB + t;
    double* rp = a.rout;
    double x0[12], x1[12];
#pragma unroll
    for (int i = 0; i < 12; ++i) {
      const int64_t row = base + 256 * i;
      const double rq = v[4 + i].x;
      double rs = 0.0;
      if (row < w) {
        __stcs(rp + row, rq);
        rs = rq;
      }
      x0[i] = rs * rs;
    }
#pragma unroll
    for (int i = 0; i < 12; ++i) {
      const int64_t row = base + kFftL + 256 * i;
      const double rq = v[4 + i].y;
      double rs = 0.0;
      if (row < w) {
        __stcs(rp + row, rq);
        rs = rq;
      }
      x1[i] = rs * rs;
    }
    if (sb + gridDim.x < nsb) {  // the next spectrum, into the registers the transform just left
      const double2* Zs = a.Z + (sb + gridDim.x) * kFftN + t;
#pragma unroll
      for (int r = 0; r < 16; ++r) v[r] = __ldcs(Zs + 256 * r);
    }
    warp_reduce12(x0, lane);
    warp_reduce12(x1, lane);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int cl = 96 * h + 8 * vi + warp;  // chunk of the superblock
      const int64_t cg = sb * kFftChunksSB + cl;
      const double xv = h ? x1[0] : x0[0];
      if (writer) {
        csB[cl] = xv;
        if (cg * kChunk < w) a.chunkB[cg] = xv;
      }
    }
    __syncthreads();
    fft_tile_sums(csB, a.tileB, sb, w);
    // csB is rewritten only after the next fft4096's barriers
  }
}

// The scores of lag q on their own (FftPassArgs::split): phase 2 of every
// superblock + the tile sums of s_q, one CTA per superblock.  It depends on
// nothing the lag's solve produces (the pending residuals, their R and the
// chunk sums of lag q - 1 are all there once the draws are done), so the sweep
// runs it on a second stream beside the solve, whose pivoted Cholesky and SVD
// occupy 16 SMs; the pass proper (transform -> r_q, B) then moves 18.7 B/row.
// Must finish before the pass of lag q starts (which overwrites chunkB).
constexpr int kFoldSB = 1;  // superblocks per CTA of k_fft_fold
__global__ void __launch_bounds__(kFftT) k_fft_fold(FftPassArgs a) {
  // One superblock per CTA.  Four consecutive ones per CTA (one folds, three only advance 192 chunk
  // sums) measured slower: the fold + pass of the instrumented C4 sweep 3.80 vs 3.42 s -- the short
  // CTAs of the non-folding superblocks are what fills the SMs between the folding CTAs' round trips.
  __shared__ double csA[2][kFftChunksSB];
  __shared__ double invRp[kFftSlots];
  const int t = threadIdx.x;
  if (t < kFftSlots) invRp[t] = t < a.npend ? 1.0 / a.Rp[t] : 0.0;
  __syncthreads();
  const int64_t nsb = (a.w + kFftSB - 1) / kFftSB;
#pragma unroll 1
  for (int j = 0; j < kFoldSB; ++j) {
    const int64_t sb = (int64_t)blockIdx.x * kFoldSB + j;
    if (sb >= nsb) break;
    const bool fold = fft_folds(a, sb);
    double oA = 0.0, oB = 0.0;
    if (!fold && t < kFftChunksSB) {
      const int64_t cg = sb * kFftChunksSB + t;
      if (cg * kChunk < a.w) {
        oA = a.chunkA[cg];
        oB = a.chunkB[cg];
      }
    }
    double* cs = csA[j & 1];  // two buffers: iteration j + 1 writes while stragglers still sum iteration j's
    fft_scores_phase(a, sb, fold, cs, invRp, oA, oB);
    __syncthreads();
    fft_tile_sums(cs, a.tileA, sb, a.w);
  }
}

}  // namespace tfk
