// Drop-in for pcs/rng.hpp (proj/include/pcs/rng.hpp:12-50): SplitMix64, the
// generator behind RandomFirstPoint and the seeded synthetic inputs. The
// device kernels carry an identical copy (csrc/device_common.cuh).
#pragma once

#include <cstdint>

namespace pcs {

class SplitMix64 {
 public:
  explicit SplitMix64(std::uint64_t seed) : state_(seed) {}

  std::uint64_t next() {
    state_ += 0x9E3779B97F4A7C15ULL;
    std::uint64_t z = state_;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
  }

  // Rejection sampling below 2^64 mod bound keeps the draw unbiased.
  std::uint64_t below(std::uint64_t bound) {
    const std::uint64_t reject_below = (0 - bound) % bound;
    std::uint64_t r = next();
    while (r < reject_below) r = next();
    return r % bound;
  }

  double unit() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
  double uniform(double lo, double hi) { return lo + (hi - lo) * unit(); }

 private:
  std::uint64_t state_;
};

}  // namespace pcs
