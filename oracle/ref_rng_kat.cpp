// Known-answer generator for the RNG, compiled directly against the
// reference's own header (proj/include/toepfit/rng.hpp, Eigen-free).
// Output: JSON on stdout, committed as tests/golden/rng_kat.json by
// oracle/make_golden.py.  TEST INFRASTRUCTURE ONLY.
#include <cstdio>
#include <cstdint>
#include <vector>

#include "toepfit/rng.hpp"

using toepfit::Rng;
using toepfit::derive_seed;

int main() {
  std::printf("{\n");
  // derive_seed table
  std::printf("  \"derive_seed\": [");
  const std::uint64_t seeds[] = {0, 1, 5, 42, 0x5c07e5u, 0xdeadbeefcafef00dull};
  const std::uint64_t tags[] = {0, 1, 2, 3, 100, 0x10001u, 0x20000u, 0x30000u, 0x5c07e5u, 0x1000u};
  bool first = true;
  for (auto s : seeds)
    for (auto t : tags) {
      std::printf("%s\n    [\"%llu\", \"%llu\", \"%llu\"]", first ? "" : ",",
                  (unsigned long long)s, (unsigned long long)t,
                  (unsigned long long)derive_seed(s, t));
      first = false;
    }
  std::printf("\n  ],\n");
  // raw draws, uniform01, normal, below
  auto dump_stream = [](const char* name, std::uint64_t seed, int count) {
    Rng r(seed);
    std::printf("  \"%s\": {\"seed\": \"%llu\", \"raw\": [", name, (unsigned long long)seed);
    for (int i = 0; i < count; ++i) std::printf("%s\"%llu\"", i ? ", " : "", (unsigned long long)r());
    Rng u(seed);
    std::printf("], \"uniform01\": [");
    for (int i = 0; i < count; ++i) std::printf("%s%.17g", i ? ", " : "", u.uniform01());
    Rng nrm(seed);
    std::printf("], \"normal\": [");
    for (int i = 0; i < count; ++i) std::printf("%s%.17g", i ? ", " : "", nrm.normal());
    Rng b(seed);
    std::printf("], \"below_1000003\": [");
    for (int i = 0; i < count; ++i)
      std::printf("%s%llu", i ? ", " : "", (unsigned long long)b.below(1000003));
    std::printf("]}");
  };
  dump_stream("stream_1", derive_seed(1, 1), 64);
  std::printf(",\n");
  dump_stream("stream_2", 0x0123456789abcdefull, 64);
  std::printf(",\n");
  dump_stream("stream_3", 42, 64);
  std::printf("\n}\n");
  return 0;
}
