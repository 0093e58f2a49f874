// pbdr/rng.hpp -- the reference's deterministic RNG at its own include path
// (proj/include/pbdr/rng.hpp:10-29): splitmix64 with the state pre-advanced
// by one increment at construction, doubles from the top 53 bits. The scene
// generators (csrc/pbdr_scene.cpp) draw from the same stream.
#pragma once

#include <cstdint>

namespace pbdr {

class Rng {
 public:
  explicit Rng(uint64_t seed) : s_(seed + kGamma) {}

  uint64_t next_u64() {
    s_ += kGamma;
    uint64_t z = s_;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  }
  double next_unit() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }  // [0, 1)
  double next_in(double lo, double hi) { return lo + (hi - lo) * next_unit(); }     // [lo, hi)

 private:
  static constexpr uint64_t kGamma = 0x9E3779B97F4A7C15ull;
  uint64_t s_;
};

}  // namespace pbdr
