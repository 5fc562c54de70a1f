// Golden-vector generator for the seeded RNG. TEST INFRASTRUCTURE ONLY.
// Compiled (oracle/Makefile target `ref`) against the UNMODIFIED reference
// header /root/reference/proj/include/traceopt/detail/rng.hpp -- the one
// hot-path-adjacent reference file that builds without Eigen.
// Output: one line per draw, "<kind> <value>", for a fixed op script, so the
// restated bae::Rng (include/bae/rng.hpp) can be pinned bit-for-bit.
#include <cinttypes>
#include <cstdio>
#include <cstdlib>

#include "traceopt/detail/rng.hpp"

int main(int argc, char** argv) {
  if (argc != 3) {
    std::fprintf(stderr, "usage: rng_golden <seed> <n_ops>\n");
    return 1;
  }
  const std::uint64_t seed = std::strtoull(argv[1], nullptr, 10);
  const int n_ops = std::atoi(argv[2]);
  traceopt::detail::Rng rng(seed);
  for (int i = 0; i < n_ops; ++i) {
    switch (i % 6) {
      case 0: std::printf("u %.17g\n", rng.uniform()); break;
      case 1: std::printf("n %.17g\n", rng.normal()); break;
      case 2: std::printf("i %" PRIu64 "\n", rng.index(1000)); break;
      case 3: std::printf("r %.17g\n", rng.uniform(-0.5, 0.5)); break;
      case 4: std::printf("n %.17g\n", rng.normal()); break;
      case 5: std::printf("i %" PRIu64 "\n", rng.index(16)); break;
    }
  }
  return 0;
}
