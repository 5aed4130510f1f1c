// Host-only probe of labsolve::Rng (include/labsolve/rng.hpp) for
// tests/test_skew_cpu.py::test_host_rng_matches_reference: stdin lines
// "seed count k0 lo0 hi0 k1 lo1 hi1 ..." -> one line of draws (uniform01 as
// its IEEE bits).
#include <cstdint>
#include <cstring>
#include <iostream>
#include <sstream>
#include <string>

#include "labsolve/rng.hpp"

int main() {
  std::string line;
  while (std::getline(std::cin, line)) {
    std::istringstream in(line);
    unsigned long long seed;
    int count;
    in >> seed >> count;
    labsolve::Rng rng(seed);
    for (int i = 0; i < count; ++i) {
      int k;
      long long lo, hi;
      in >> k >> lo >> hi;
      unsigned long long v;
      if (k == 0) {
        v = rng.bits64();
      } else if (k == 1) {
        v = static_cast<unsigned long long>(rng.uniform_int(lo, hi));
      } else {
        const double d = rng.uniform01();
        std::memcpy(&v, &d, sizeof v);
      }
      std::cout << v << (i + 1 < count ? ' ' : '\n');
    }
  }
  return 0;
}
