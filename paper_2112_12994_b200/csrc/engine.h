// engine.h -- host-side context of the B200 toepfit engine (C++).
#pragma once

#include <cuda_runtime.h>

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
  void need(size_t count);
  void release();
  T* get() const { return p; }
};

struct SolveBufs {
  DBuf<double> W, G, RA, RB, RC, SA, SB, SC, T, S0, S1, Q1, Q2;
  DBuf<int> flags, tickets;
};

}  // namespace tfe

struct tf_context {
  int device = 0;
  cudaStream_t stream = nullptr;
  std::string err;
  int sm_count = 148;
  // series
  tfe::DBuf<double> y;
  int64_t n = 0;
  // LSAR state
  tfe::DBuf<double> s, r, chunkA, chunkB, tileA, tileB, OT, scal, Rhist, Shist, phi, coefs, taus;
  tfe::DBuf<int64_t> idx, fidx, idx_hist;
  tfe::DBuf<double> wts, fw, w_hist;
  tfe::DBuf<int> status, method;
  tfe::SolveBufs sb;
  // RH state
  tfe::DBuf<double> rh_scores, rh_approx, rh_approx2, rh_M, rh_G;
  tfe::DBuf<int64_t> rh_lvl, rh_tmp, rh_picked;
  tfe::DBuf<uint64_t> rh_keys, rh_keys2;
  tfe::DBuf<unsigned char> rh_cub;
  std::vector<cudaEvent_t> events;
  std::vector<cudaEvent_t> pev;  // phase events (2 per lag)
  int64_t launches = 0;
};
