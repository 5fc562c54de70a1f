// Deterministic random source shared by the synthetic-scene generator and the
// test oracle. Restates the reference's seeded generator
// (traceopt::detail::Rng, /root/reference/proj/include/traceopt/detail/rng.hpp:12-48):
// a 64-bit Mersenne twister whose raw words are turned into doubles and
// normals by hand-written transforms, so a seed pins the exact value stream
// regardless of the C++ standard library's distribution implementations.
//
// Pinned against the reference header itself: oracle/ref/rng_golden.cpp is
// compiled against the unmodified reference rng.hpp (oracle/Makefile, target
// _ref) and its stream is committed as tests/golden/rng_streams.json.
#pragma once

#include <cmath>
#include <cstdint>
#include <random>

namespace bae {

class Rng {
 public:
  explicit Rng(std::uint64_t seed) : mt_(seed) {}

  // [0, 1): top 53 bits of one engine word scaled by 2^-53 (rng.hpp:17-19).
  double uniform() { return static_cast<double>(mt_() >> 11) * 0x1.0p-53; }

  double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }

  // Polar-free Box-Muller pair; the sine branch is kept for the next call
  // (rng.hpp:24-37). u1 is redrawn while it is exactly zero.
  double normal() {
    if (cached_) {
      cached_ = false;
      return cache_;
    }
    double a = uniform();
    while (a <= 0.0) a = uniform();
    const double b = uniform();
    const double radius = std::sqrt(-2.0 * std::log(a));
    const double angle = 2.0 * M_PI * b;
    cache_ = radius * std::sin(angle);
    cached_ = true;
    return radius * std::cos(angle);
  }

  double normal(double mean, double sigma) { return mean + sigma * normal(); }

  // Modulo reduction of one raw word (rng.hpp:42).
  std::uint64_t index(std::uint64_t n) { return mt_() % n; }

 private:
  std::mt19937_64 mt_;
  double cache_ = 0.0;
  bool cached_ = false;
};

}  // namespace bae
