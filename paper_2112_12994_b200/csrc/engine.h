// engine.h -- host-side context of the B200 toepfit engine (C++).
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>

#include <cstdint>
#include <string>
#include <vector>

#include "../../include/toepfit_b200.h"

namespace tfe {

struct TfError {
  tf_status code;
  std::string msg;
};

// grow-only device buffer
template <class T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
  DBuf() = default;
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  ~DBuf() { release(); }  // every buffer of a context is freed by tf_destroy's delete
  void need(size_t count);
  void release();
  T* get() const { return p; }
};

// captured launch sequence of a sweep shape (see lsar_sweep)
struct GraphCache {
  cudaGraphExec_t exec = nullptr;
  uint64_t gen = 0;
  int64_t w = 0, c = 0, launches = 0;
  int p_bar = 0, mode = 0, seen = 0;
};

struct SolveBufs {
  DBuf<double> W, G, RA, RB, RC, SA, SB, SC, T, S0, S1, Q1, Q2, M, RI;
  DBuf<int> flags;
  // rank-revealing solve (k_exact.cuh): double-double Gram partials and
  // planes, pivoted factor, SVD matrix / singular values / partial solutions
  DBuf<double> Wdd, Gh, Gl, Rh, Rl, Dd, Nsv, sig, xpart, tolv, cn, cnp;
  DBuf<double> Gloc, Gg;  // row-sharded sweeps: this shard's Gram partial [2][K*K], the allgathered partials
  DBuf<int> perm, svdf;
  // INT8 tensor-core Gram (k_i8gram.cuh): pre-tiled digit planes, column
  // exponents, int32 product tiles, the tile lists of every plane width
  DBuf<unsigned char> i8D;
  DBuf<int> i8E, i8P, i8tiles, i8tof;
  std::vector<int> i8_tile_off, i8_tof_off, i8_ntiles;  // per nbs (host copies of the table layout)
};

}  // namespace tfe

struct tf_context {
  int device = 0;
  cudaStream_t stream = nullptr;
  // second stream (lowest priority) + fork / join events: the FFT lags' score update (k_fft_fold)
  // runs beside the lag's solve (engine.cu, lsar_sweep)
  cudaStream_t side = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  int fft_split = 1;
  std::string err;
  int sm_count = 148;
  int smem_optin_max = 232448;  // cudaDevAttrMaxSharedMemoryPerBlockOptin
  // series
  tfe::DBuf<double> y;
  int64_t n = 0;
  // LSAR state
  tfe::DBuf<double> s, r, chunkA, chunkB, tileA, tileB, OT, scal, Rhist, Shist, phi, coefs, taus;
  tfe::DBuf<int> guide;  // draw guide table (k_lag_scan)
  tfe::DBuf<double> scan_part, scan_boff;  // multi-CTA scan of long windows: block totals, block prefixes
  tfe::DBuf<double> srht_X, srht_D;  // SRHT: transform batch, sampled dense system
  tfe::DBuf<int64_t> srht_draws;
  tfe::DBuf<int> srht_reject;
  tfe::DBuf<int64_t> idx, fidx, idx_hist;
  tfe::DBuf<double> wts, fw, w_hist;
  tfe::DBuf<int> status, method, rank, sweeps;
  tfe::SolveBufs sb;
  // RH state
  tfe::DBuf<int> rh_J, rh_cnt, rh_start, rh_fill, rh_bk, rh_pick, rh_ok, rh_flag;
  tfe::DBuf<long long> rh_tsum;
  tfe::DBuf<int64_t> rh_lvl, rh_aidx, rh_sidx, rh_fup;
  tfe::DBuf<double> rh_scores, rh_aw, rh_sw, rh_fupw, rh_ones, rh_norm, rh_Gp, rh_H0, rh_W, rh_S,
      rh_phis, rh_rest, rh_part;
  // row-sharded LSAR sweep (tf_lsar_sweep_sharded): NCCL communicator, the
  // allgathered shard sums, this shard's CDF segment, its compacted draws
  ncclComm_t comm = nullptr;
  int nc_world = 1, nc_rank = 0;
  tfe::DBuf<double> sh_part, sh_gath, sh_par, sh_wts;
  tfe::DBuf<int64_t> sh_idx;
  tfe::DBuf<int> sh_dummy;
  tfe::DBuf<double> scratch;  // blocked Cholesky (cholinv_big) trace scratch
  // batched LSAR sweeps of equal-shape series (tf_lsar_sweep_batch)
  tfe::DBuf<double> bt_y, bt_s, bt_r, bt_cA, bt_cB, bt_tA, bt_tB, bt_OT, bt_scal, bt_Rh, bt_Sh, bt_phi,
      bt_coefs, bt_taus, bt_wts, bt_S0, bt_S1, bt_fw;
  tfe::DBuf<int64_t> bt_idx, bt_fidx;
  tfe::DBuf<uint64_t> bt_seed;
  tfe::DBuf<int> bt_status, bt_fb, bt_guide, bt_method;
  tfe::DBuf<unsigned long long> fincheck;  // upload validation
  cudaEvent_t ev_begin = nullptr, ev_end = nullptr;  // span of the last sweep
  tfe::GraphCache lsar_graph, rh_graph;
  tfe::DBuf<uint64_t> seedtab;
  bool no_graphs = false;
  // FFT pass (k_fft.cuh): series spectra of this sweep, the lag's filter
  // spectrum, twiddle tables; pass_mode 0 auto (FFT for lags >= fft_minq),
  // 1 direct FIR only, 2 FFT at every lag >= 1
  tfe::DBuf<double2> fftZ, fftH, fftTw, fftTwH, fftTwL;  // fftTwH/L: W_4096^e, e < 4096, double-double
  tfe::DBuf<unsigned long long> ymax;  // max |y| of the resident series (bit pattern), per sweep
  int pass_mode = 0, fft_minq = 0, fft_minlags = 0;
  int fft_slots = 4;                // deferred folding groups of the FFT pass (k_fft.cuh kFftSlots; 1 = fold per lag)
  tfe::DBuf<double> fft_rslot[4];   // residual slots 1..4 (slot 0 is r; K groups use K + 1 slots)
  int gram_mode = 0;  // 0 auto (INT8 tensor-core Gram above a work threshold), 1 double-double CUDA cores, 2 INT8 whenever c fits
  std::vector<cudaEvent_t> events;
  std::vector<cudaEvent_t> pev;  // phase events (2 per lag)
  int64_t launches = 0;
  int step_p = 0;     // lag of the LsarDriver state resident in s / r (tf_lsar_step), 0: none
  int64_t step_w = 0;
};
