// toepfit_b200.hpp -- header-only C++17 host API over the C ABI
// (include/toepfit_b200.h), mirroring the reference's fit surface in
// namespace toepfit (proj/include/toepfit):
//
//   TimeSeries                series.hpp:16-31 (shared immutable storage)
//   UsageError / DataError /  errors.hpp:12-29 (thrown from the C-ABI status)
//     NumericalError
//   PACFResult, PacfMethod    toeplitz.hpp:64-68
//   FitResult                 lsar.hpp:28-35 (std::vector instead of Eigen::VectorXd)
//   RHConfig                  repeated_halving.hpp:56-65 (defaults / validate)
//   lsar_fit                  lsar.hpp:89
//   rh_fit (5- and 4-arg)     repeated_halving.hpp:97-99
//   LeverageState, LsarDriver lsar.hpp:17-23, 65-84 (first_lag / advance / row_count)
//   RowSource, DenseRowSource, repeated_halving.hpp:17-91
//     GaussianSketch, SpectralApprox, generalized_leverage, repeated_halving
//   select_order              toeplitz.hpp:100
//
// One device context per host thread (created lazily on device 0, or bound
// with toepfit::gpu::use_device); the reference is single-threaded and
// distinct fits may run concurrently on distinct threads.
// Nothing here computes on the CPU: without a CUDA device every call throws
// toepfit::gpu::CudaError.
#ifndef TOEPFIT_B200_HPP
#define TOEPFIT_B200_HPP

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "toepfit_b200.h"

namespace toepfit {

class UsageError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class DataError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class NumericalError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};

namespace gpu {
class CudaError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
}  // namespace gpu

class TimeSeries {
 public:
  explicit TimeSeries(std::vector<double> values, std::string label = "")
      : values_(std::make_shared<const std::vector<double>>(std::move(values))), label_(std::move(label)) {
    if (values_->empty()) throw DataError("series must contain at least one value");
    for (std::size_t i = 0; i < values_->size(); ++i)
      if (!std::isfinite((*values_)[i]))
        throw DataError("series value at position " + std::to_string(i) + " is not finite");
  }
  const std::vector<double>& values() const { return *values_; }
  std::size_t size() const { return values_->size(); }
  const std::string& label() const { return label_; }
  std::shared_ptr<const std::vector<double>> storage() const { return values_; }

 private:
  std::shared_ptr<const std::vector<double>> values_;
  std::string label_;
};

enum class PacfMethod { exact, lsar, rh, srht };

struct PACFResult {
  std::vector<double> taus;
  double bound = 0.0;
  PacfMethod method = PacfMethod::exact;
};

struct FitResult {
  int p_star = 0;
  std::vector<double> coefficients;
  PACFResult pacf;
  std::vector<double> per_lag_seconds;
  std::vector<std::vector<double>> per_lag_coefficients;
  double upfront_seconds = 0.0;
};

struct RHConfig {
  std::int64_t base_threshold = 0;
  std::int64_t sample_count = 0;
  std::int64_t gaussian_rows = 0;
  std::uint64_t seed = 0;

  static RHConfig defaults(std::int64_t n, std::int64_t k, std::int64_t c, std::uint64_t seed) {
    RHConfig r;
    const std::int64_t logk = (std::int64_t)std::ceil(std::log((double)k + 1.0));
    r.base_threshold = c > 10 * k * logk ? c : 10 * k * logk;
    r.sample_count = c;
    r.gaussian_rows = (std::int64_t)std::ceil(8.0 * std::log((double)(n > 2 ? n : 2)));
    r.seed = seed;
    return r;
  }
  void validate() const {
    if (sample_count < 1) throw UsageError("sample count must be positive");
    if (base_threshold < sample_count) throw UsageError("base threshold below sample count");
    if (gaussian_rows < 1) throw UsageError("need at least one sketch row");
  }
};

namespace gpu {

inline void raise(tf_status st, const tf_context* ctx) {
  const std::string msg = ctx ? tf_last_error(ctx) : std::string("no CUDA device");
  switch (st) {
    case TF_OK: return;
    case TF_USAGE: throw UsageError(msg);
    case TF_DATA: throw DataError(msg);
    case TF_NUMERICAL: throw NumericalError(msg);
    default: throw CudaError(msg);
  }
}

// per-thread device context with the last uploaded series cached by identity
struct Context {
  tf_context* ctx = nullptr;
  int device = 0;
  const std::vector<double>* cached = nullptr;
  std::shared_ptr<const std::vector<double>> keep;
  ~Context() {
    if (ctx) tf_destroy(ctx);
  }
  tf_context* get() {
    if (!ctx) {
      tf_opts o{device, 0};
      const tf_status st = tf_create(&o, &ctx);
      if (st != TF_OK) {
        ctx = nullptr;
        raise(st == TF_USAGE ? TF_USAGE : TF_CUDA, nullptr);
      }
    }
    return ctx;
  }
  void upload(const TimeSeries& s) {
    tf_context* c = get();
    if (cached == &s.values() && keep == s.storage()) return;
    cached = nullptr;  // a failed upload leaves no resident series: force the next upload
    keep.reset();
    raise(tf_upload_series(c, s.values().data(), (int64_t)s.size()), c);
    cached = &s.values();
    keep = s.storage();
  }
};

inline Context& context() {
  thread_local Context c;
  return c;
}

inline void use_device(int device) {
  Context& c = context();
  if (c.ctx && c.device != device) {
    tf_destroy(c.ctx);
    c.ctx = nullptr;
    c.cached = nullptr;
    c.keep.reset();
  }
  c.device = device;
}

inline FitResult finish(PacfMethod m, int p_bar, std::int64_t c, const std::vector<double>& taus,
                        const std::vector<double>& packed, std::vector<double> secs, int p_star,
                        double upfront) {
  FitResult f;
  f.pacf.taus = taus;
  f.pacf.bound = 1.96 / std::sqrt((double)c);
  f.pacf.method = m;
  f.per_lag_seconds = std::move(secs);
  f.p_star = p_star;
  f.upfront_seconds = upfront;
  std::size_t off = 0;
  for (int p = 1; p <= p_bar; ++p) {
    f.per_lag_coefficients.emplace_back(packed.begin() + off, packed.begin() + off + p);
    off += p;
  }
  if (p_star > 0) f.coefficients = f.per_lag_coefficients[p_star - 1];
  return f;
}

}  // namespace gpu

inline FitResult lsar_fit(const TimeSeries& series, int p_bar, std::int64_t c, std::uint64_t seed) {
  gpu::Context& g = gpu::context();
  tf_context* ctx = g.get();
  g.upload(series);
  const int pb = p_bar > 0 ? p_bar : 1;
  std::vector<double> taus(pb), packed((std::size_t)pb * (pb + 1) / 2), secs(pb);
  int p_star = 0;
  gpu::raise(tf_lsar_sweep(ctx, p_bar, c, seed, nullptr, taus.data(), packed.data(), secs.data(), &p_star),
             ctx);
  return gpu::finish(PacfMethod::lsar, p_bar, c, taus, packed, std::move(secs), p_star, 0.0);
}

// State of the lag recursion after the compressed solve at lag p
// (lsar.hpp:17-23; std::vector instead of Eigen::VectorXd).
struct LeverageState {
  int p = 0;
  std::int64_t m = 0;
  std::vector<double> scores;        // approximate leverage, length m - p
  std::vector<double> residuals;     // residuals of the lag-p compressed fit
  std::vector<double> coefficients;  // compressed phi at lag p
};

// LsarDriver (lsar.hpp:65-84): the recursion one lag at a time on the GPU
// (tf_lsar_step).  Like the reference, a state is a value: advance() uploads
// its scores and residuals (the Python mirror continues from the device-resident
// vectors when handed the state it just returned).
class LsarDriver {
 public:
  LsarDriver(const TimeSeries& series, int p_bar, std::int64_t c, std::uint64_t seed)
      : series_(series), p_bar_(p_bar), c_(c), seed_(seed) {
    if (p_bar < 1) throw UsageError("maximum lag must be at least 1");  // lsar.cpp:55-64
    if (series.size() <= static_cast<std::size_t>(p_bar) + 1)
      throw DataError("series too short for maximum lag " + std::to_string(p_bar));
    if (c < p_bar) throw UsageError("sample count below maximum lag");
    w_ = static_cast<std::int64_t>(series.size()) - p_bar;
  }
  LeverageState first_lag() const { return step(1, nullptr); }
  LeverageState advance(const LeverageState& state) const {
    if (state.p < 1 || state.p >= p_bar_) throw UsageError("cannot advance past maximum lag");  // lsar.cpp:90
    if (state.scores.size() != static_cast<std::size_t>(w_) || state.residuals.size() != static_cast<std::size_t>(w_))
      throw UsageError("state vectors must hold row_count() values");
    return step(state.p + 1, &state);
  }
  // window system for lag p: the first n - p_bar + p observations (lsar.cpp:66-68)
  std::int64_t window_length(int p) const { return w_ + p; }
  std::int64_t row_count() const { return w_; }

 private:
  LeverageState step(int p, const LeverageState* prev) const {
    gpu::Context& g = gpu::context();
    tf_context* ctx = g.get();
    g.upload(series_);
    LeverageState st;
    st.p = p;
    st.m = w_ + p;
    st.scores.resize(static_cast<std::size_t>(w_));
    st.residuals.resize(static_cast<std::size_t>(w_));
    st.coefficients.resize(static_cast<std::size_t>(p));
    int method = 0;
    gpu::raise(tf_lsar_step(ctx, p_bar_, c_, seed_, p, prev ? prev->scores.data() : nullptr,
                            prev ? prev->residuals.data() : nullptr, st.scores.data(), st.residuals.data(),
                            st.coefficients.data(), &method),
               ctx);
    return st;
  }

  const TimeSeries& series_;
  int p_bar_;
  std::int64_t c_;
  std::uint64_t seed_;
  std::int64_t w_ = 0;
};

// ---- Repeated Halving over a general row source (repeated_halving.hpp:17-91) ----
// RowSource: an n x k matrix that may never exist in memory; gather() fills
// out (idx.size() x k, row-major) with rows idx[t].
class RowSource {
 public:
  virtual ~RowSource() = default;
  virtual std::int64_t rows() const = 0;
  virtual std::int64_t cols() const = 0;
  virtual void gather(const std::vector<std::int64_t>& idx, std::vector<double>& out) const = 0;
};

class DenseRowSource final : public RowSource {
 public:
  // a: rows x cols, row-major
  DenseRowSource(std::vector<double> a, std::int64_t rows, std::int64_t cols)
      : a_(std::move(a)), rows_(rows), cols_(cols) {}
  std::int64_t rows() const override { return rows_; }
  std::int64_t cols() const override { return cols_; }
  void gather(const std::vector<std::int64_t>& idx, std::vector<double>& out) const override {
    out.resize(idx.size() * (std::size_t)cols_);
    for (std::size_t t = 0; t < idx.size(); ++t)
      for (std::int64_t j = 0; j < cols_; ++j) out[t * cols_ + j] = a_[(std::size_t)(idx[t] * cols_ + j)];
  }

 private:
  std::vector<double> a_;
  std::int64_t rows_, cols_;
};

struct GaussianSketch {
  std::int64_t rows = 0;
  std::uint64_t seed = 0;
};

struct SpectralApprox {
  std::vector<double> rows;  // sample_count x k, row-major
  int levels = 0;
  std::int64_t sample_count = 0;
};

// leverage of the rows of C (rows x k, row-major) through B's column space
inline std::vector<double> generalized_leverage(const std::vector<double>& c_rows, std::int64_t rows,
                                                const std::vector<double>& b, std::int64_t brows, std::int64_t k,
                                                const GaussianSketch* sketch = nullptr) {
  gpu::Context& g = gpu::context();
  tf_context* ctx = g.get();
  std::vector<double> out((std::size_t)(rows > 0 ? rows : 1));
  gpu::raise(tf_generalized_leverage(ctx, c_rows.data(), rows, k, b.data(), brows, k, sketch ? sketch->rows : 0,
                                     sketch ? sketch->seed : 0, out.data()),
             ctx);
  out.resize((std::size_t)rows);
  return out;
}

inline SpectralApprox repeated_halving(const RowSource& x, const RHConfig& config) {
  config.validate();
  gpu::Context& g = gpu::context();
  tf_context* ctx = g.get();
  struct Shim {
    const RowSource* src;
    std::vector<std::int64_t> ids;
    std::vector<double> buf;
  } shim{&x, {}, {}};
  auto cb = [](void* user, const int64_t* idx, int64_t count, double* out) {
    Shim* s = static_cast<Shim*>(user);
    s->ids.assign(idx, idx + count);
    s->src->gather(s->ids, s->buf);
    std::copy(s->buf.begin(), s->buf.end(), out);
  };
  const std::int64_t n = x.rows(), k = x.cols();
  const std::int64_t cap = std::max<std::int64_t>({config.sample_count, config.base_threshold, std::int64_t(1)});
  SpectralApprox a;
  a.rows.resize((std::size_t)(cap * k));
  const tf_rh_cfg cfg{config.base_threshold, config.sample_count, config.gaussian_rows, config.seed};
  std::int64_t ar = 0;
  gpu::raise(tf_repeated_halving(ctx, n, k, cb, &shim, &cfg, a.rows.data(), cap, &ar, &a.levels), ctx);
  a.rows.resize((std::size_t)(ar * k));
  a.sample_count = ar;
  return a;
}

// Many independent LSAR fits in one batched sweep (tf_lsar_sweep_batch): fit b
// = lsar_fit(series[b], p_bar, c, seeds[b]); equal-length series, p_bar <= 63.
// The reference's run_compare / run_sweep repetition loops (bench.cpp:183-188,
// 221-228) pass the same series for every seed.  Throws the first failing
// fit's exception.  per_lag_seconds: the batch's per-lag time / fits.
inline std::vector<FitResult> lsar_fit_batch(const std::vector<TimeSeries>& series, int p_bar, std::int64_t c,
                                             const std::vector<std::uint64_t>& seeds) {
  if (series.size() != seeds.size() || series.empty()) throw UsageError("one seed per series, at least one fit");
  const std::size_t n = series[0].size();
  std::vector<double> y;
  y.reserve(n * series.size());
  for (const TimeSeries& s : series) {
    if (s.size() != n) throw UsageError("batched fits need equal-length series");
    y.insert(y.end(), s.values().begin(), s.values().end());
  }
  gpu::Context& g = gpu::context();
  tf_context* ctx = g.get();
  g.cached = nullptr;  // a re-run fit replaces the resident series
  const std::int64_t B = (std::int64_t)series.size();
  const int pb = p_bar > 0 ? p_bar : 1;
  const std::size_t nc = (std::size_t)pb * (pb + 1) / 2;
  std::vector<double> taus((std::size_t)B * pb), packed((std::size_t)B * nc), secs(pb);
  std::vector<int> p_star((std::size_t)B), status((std::size_t)(3 * B));
  gpu::raise(tf_lsar_sweep_batch(ctx, y.data(), (std::int64_t)n, B, (std::int64_t)n, p_bar, c, seeds.data(),
                                 nullptr, nullptr, taus.data(), packed.data(), secs.data(), p_star.data(),
                                 status.data()),
             ctx);
  for (double& s : secs) s /= (double)B;
  std::vector<FitResult> out;
  for (std::int64_t b = 0; b < B; ++b) {
    if (status[3 * b]) {
      const std::string what = "fit " + std::to_string(b) + " failed at lag " + std::to_string(status[3 * b + 1]);
      if (status[3 * b] == 1) throw UsageError(what);
      if (status[3 * b] == 2) throw DataError(what);
      throw NumericalError(what);
    }
    out.push_back(gpu::finish(PacfMethod::lsar, p_bar, c,
                              std::vector<double>(taus.begin() + b * pb, taus.begin() + (b + 1) * pb),
                              std::vector<double>(packed.begin() + b * nc, packed.begin() + (b + 1) * nc), secs,
                              p_star[b], 0.0));
  }
  return out;
}

inline FitResult rh_fit(const TimeSeries& series, int p_bar, std::int64_t c, const RHConfig* config,
                        std::uint64_t seed) {
  gpu::Context& g = gpu::context();
  tf_context* ctx = g.get();
  g.upload(series);
  tf_rh_cfg cfg{};
  if (config) {
    config->validate();
    cfg = tf_rh_cfg{config->base_threshold, config->sample_count, config->gaussian_rows, config->seed};
  }
  const int pb = p_bar > 0 ? p_bar : 1;
  std::vector<double> taus(pb), packed((std::size_t)pb * (pb + 1) / 2), secs(pb);
  double upfront = 0.0;
  int p_star = 0;
  gpu::raise(tf_rh_sweep(ctx, p_bar, c, config ? &cfg : nullptr, seed, nullptr, taus.data(), packed.data(),
                         secs.data(), &upfront, &p_star),
             ctx);
  return gpu::finish(PacfMethod::rh, p_bar, c, taus, packed, std::move(secs), p_star, upfront);
}

inline FitResult rh_fit(const TimeSeries& series, int p_bar, std::int64_t c, std::uint64_t seed) {
  return rh_fit(series, p_bar, c, nullptr, seed);
}

// exact per-lag OLS (bench.cpp:27-48); bound 1.96 / sqrt(n - p_bar)
inline FitResult exact_fit(const TimeSeries& series, int p_bar) {
  gpu::Context& g = gpu::context();
  tf_context* ctx = g.get();
  g.upload(series);
  const int pb = p_bar > 0 ? p_bar : 1;
  std::vector<double> taus(pb), packed((std::size_t)pb * (pb + 1) / 2), secs(pb);
  int p_star = 0;
  gpu::raise(tf_exact_sweep(ctx, p_bar, taus.data(), packed.data(), secs.data(), &p_star), ctx);
  FitResult f = gpu::finish(PacfMethod::exact, p_bar, 1, taus, packed, std::move(secs), p_star, 0.0);
  f.pacf.bound = 1.96 / std::sqrt((double)series.size() - p_bar);
  return f;
}

// subsampled randomized Hadamard transform fit (bench.cpp:50-72)
inline FitResult srht_fit(const TimeSeries& series, int p_bar, std::int64_t c, std::uint64_t seed) {
  gpu::Context& g = gpu::context();
  tf_context* ctx = g.get();
  g.upload(series);
  const int pb = p_bar > 0 ? p_bar : 1;
  std::vector<double> taus(pb), packed((std::size_t)pb * (pb + 1) / 2), secs(pb);
  int p_star = 0;
  gpu::raise(tf_srht_sweep(ctx, p_bar, c, seed, taus.data(), packed.data(), secs.data(), &p_star), ctx);
  return gpu::finish(PacfMethod::srht, p_bar, c, taus, packed, std::move(secs), p_star, 0.0);
}

inline int select_order(const PACFResult& pacf) {
  return tf_select_order(pacf.taus.data(), (int)pacf.taus.size(), pacf.bound);
}

}  // namespace toepfit

#endif  // TOEPFIT_B200_HPP
