// rng.hpp — drop-in for /root/reference/proj/include/labsolve/rng.hpp:10-28.
//
// Same class, same draws: std::mt19937_64 seeded once, libstdc++ 13's
// uniform_int_distribution<long long> (Lemire, 128-bit product) and
// generate_canonical<double> (one draw). The engine state is a plain
// labs_rng_state so the device kernels can continue the exact stream the
// caller holds (include/labs_b200.h) and hand it back advanced.
#pragma once

#include <cstdint>

#include "labs_b200.h"

namespace labsolve {

class Rng {
 public:
  explicit Rng(std::uint64_t seed);

  std::uint64_t bits64();
  // Uniform integer on [lo, hi], both ends inclusive.
  long long uniform_int(long long lo, long long hi);
  // Uniform real on [0, 1).
  double uniform01();

  // B200 extension: the engine state shared with the device kernels.
  labs_rng_state& state() { return st_; }
  const labs_rng_state& state() const { return st_; }

 private:
  labs_rng_state st_;
};

}  // namespace labsolve
