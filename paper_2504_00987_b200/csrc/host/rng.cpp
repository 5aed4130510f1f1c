// Host side of the Rng contract (rng.hpp). The engine is MT19937-64; the
// distributions follow libstdc++ 13 (uniform_int_dist.h:255-281,
// random.tcc:3346-3381) so a stream can move between host and device.
#include "labsolve/rng.hpp"

#include <cmath>

namespace labsolve {
namespace {

constexpr int kN = 312, kM = 156;
constexpr std::uint64_t kUpper = 0xFFFFFFFF80000000ULL, kLower = 0x7FFFFFFFULL;
constexpr std::uint64_t kMatrix = 0xB5026F5AA96619E9ULL;

inline std::uint64_t mix(std::uint64_t a, std::uint64_t b, std::uint64_t c) {
  const std::uint64_t x = (a & kUpper) | (b & kLower);
  return c ^ (x >> 1) ^ ((x & 1ULL) ? kMatrix : 0ULL);
}

void regenerate(labs_rng_state& s) {
  std::uint64_t* m = s.mt;
  for (int i = 0; i < kN; ++i) {
    const int nxt = (i + 1) % kN;
    const int far = (i + kM) % kN;
    m[i] = mix(m[i], m[nxt], m[far]);
  }
  s.idx = 0;
}

}  // namespace

Rng::Rng(std::uint64_t seed) { labs_rng_seed(seed, &st_); }

std::uint64_t Rng::bits64() {
  if (st_.idx >= kN) regenerate(st_);
  std::uint64_t y = st_.mt[st_.idx++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  return y ^ (y >> 43);
}

long long Rng::uniform_int(long long lo, long long hi) {
  const std::uint64_t span =
      static_cast<std::uint64_t>(hi) - static_cast<std::uint64_t>(lo) + 1ULL;
  if (span == 0) return static_cast<long long>(bits64());
  unsigned __int128 p = static_cast<unsigned __int128>(bits64()) * span;
  if (static_cast<std::uint64_t>(p) < span) {
    const std::uint64_t floor_ = (0ULL - span) % span;
    while (static_cast<std::uint64_t>(p) < floor_)
      p = static_cast<unsigned __int128>(bits64()) * span;
  }
  return static_cast<long long>(static_cast<std::uint64_t>(lo) +
                                static_cast<std::uint64_t>(p >> 64));
}

double Rng::uniform01() {
  const double d = static_cast<double>(bits64()) * 0x1p-64;
  return d < 1.0 ? d : std::nextafter(1.0, 0.0);
}

}  // namespace labsolve
