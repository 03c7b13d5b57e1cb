// C++ host-API check (include/toepfit_b200.hpp): the reference's call shapes
// (toepfit::lsar_fit / rh_fit / select_order / TimeSeries / exception types)
// on a GPU.  Reads the series (raw little-endian fp64) from argv[1], prints one
// JSON object; tests/test_cpp_api.py compares it with the Python API.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iterator>
#include <string>
#include <vector>

#include "toepfit_b200.hpp"

static void print_fit(const char* name, const toepfit::FitResult& f, bool comma) {
  std::printf("\"%s\": {\"p_star\": %d, \"upfront\": %.17g, \"taus\": [", name, f.p_star, f.upfront_seconds);
  for (std::size_t i = 0; i < f.pacf.taus.size(); ++i)
    std::printf("%s%.17g", i ? ", " : "", f.pacf.taus[i]);
  std::printf("], \"select\": %d}%s\n", toepfit::select_order(f.pacf), comma ? "," : "");
}

int main(int argc, char** argv) {
  if (argc < 5) {
    std::fprintf(stderr, "usage: %s series.bin p_bar c seed\n", argv[0]);
    return 2;
  }
  std::ifstream in(argv[1], std::ios::binary);
  std::vector<char> raw((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
  std::vector<double> y(raw.size() / sizeof(double));
  std::memcpy(y.data(), raw.data(), y.size() * sizeof(double));
  const int p_bar = std::stoi(argv[2]);
  const long long c = std::stoll(argv[3]);
  const unsigned long long seed = std::stoull(argv[4]);
  toepfit::TimeSeries series(std::move(y), "cpp");
  std::printf("{\n");
  print_fit("lsar", toepfit::lsar_fit(series, p_bar, c, seed), true);
  print_fit("rh", toepfit::rh_fit(series, p_bar, c, seed), true);
  print_fit("srht", toepfit::srht_fit(series, p_bar, c, seed), true);
  print_fit("exact", toepfit::exact_fit(series, p_bar), true);
  {  // batched: two seeds over the same series
    const auto fits = toepfit::lsar_fit_batch({series, series}, p_bar, c, {seed, seed + 1});
    print_fit("batch0", fits[0], true);
    print_fit("batch1", fits[1], true);
  }
  {  // LsarDriver (lsar.hpp:65-84): first_lag / advance, replay determinism
    toepfit::LsarDriver drv(series, p_bar, c, seed);
    const toepfit::LeverageState s1 = drv.first_lag();
    const toepfit::LeverageState s2 = drv.advance(s1);
    const toepfit::LeverageState r2 = drv.advance(drv.first_lag());
    double ssum = 0.0;
    for (double v : s2.scores) ssum += v;
    std::printf("\"driver\": {\"rows\": %lld, \"m1\": %lld, \"m2\": %lld, \"p2\": %d, \"ssum2\": %.17g, "
                "\"replay\": %d, \"phi2\": [%.17g, %.17g]},\n",
                (long long)drv.row_count(), (long long)s1.m, (long long)s2.m, s2.p, ssum,
                r2.coefficients == s2.coefficients ? 1 : 0, s2.coefficients[0], s2.coefficients[1]);
  }
  {  // Repeated Halving over a dense row source (repeated_halving.hpp:17-91)
    const std::int64_t rows = 512, k = 6;
    std::vector<double> a((std::size_t)(rows * k));
    for (std::size_t i = 0; i < a.size(); ++i) a[i] = std::sin(0.37 * (double)i) + 0.01 * (double)(i % 17);
    toepfit::DenseRowSource src(a, rows, k);
    toepfit::RHConfig cfg;
    cfg.base_threshold = 128;
    cfg.sample_count = 128;
    cfg.gaussian_rows = 48;
    cfg.seed = 3;
    const toepfit::SpectralApprox ap = toepfit::repeated_halving(src, cfg);
    const std::vector<double> lev = toepfit::generalized_leverage(a, rows, a, rows, k);
    double lsum = 0.0;
    for (double v : lev) lsum += v;
    std::printf("\"rowsource\": {\"levels\": %d, \"rows\": %lld, \"lev_sum\": %.17g},\n", ap.levels,
                (long long)ap.sample_count, lsum);
  }
  // error mapping (errors.hpp:12-29 types)
  int usage = 0, data = 0, numerical = 0;
  try {
    toepfit::lsar_fit(series, p_bar, p_bar - 1, seed);
  } catch (const toepfit::UsageError&) {
    usage = 1;
  }
  try {
    toepfit::TimeSeries empty(std::vector<double>{});
  } catch (const toepfit::DataError&) {
    data = 1;
  }
  try {
    std::vector<double> g(64);
    for (int t = 0; t < 64; ++t) g[t] = std::ldexp(1.0, -t);  // 0.5^t: zero residual (test_lsar.cpp:160-169)
    toepfit::lsar_fit(toepfit::TimeSeries(g), 2, 20, 1);
  } catch (const toepfit::NumericalError&) {
    numerical = 1;
  }
  std::printf("\"errors\": {\"usage\": %d, \"data\": %d, \"numerical\": %d}\n}\n", usage, data, numerical);
  return 0;
}
