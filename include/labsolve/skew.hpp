// skew.hpp — drop-in for /root/reference/proj/include/labsolve/skew.hpp:10-40.
// Distance from skew-symmetry of found sequences (post-hoc analysis, off the
// search path): host code, O(n^2) per rotation, same evaluation order and
// budget accounting as the reference so `evaluations` match.
#pragma once

#include <cstdint>

#include "labsolve/sequence.hpp"

namespace labsolve {

Sequence rot(const Sequence& s, int count);
Sequence ins(const Sequence& s, int gap, int spin);
Sequence del(const Sequence& s, int pos);
int n_non_skew(const Sequence& s);

struct DeviationResult {
  int value = -1;
  bool budget_exceeded = false;
  std::uint64_t evaluations = 0;
};

DeviationResult deviation(const Sequence& s, std::uint64_t budget = 0);
DeviationResult deviation_with_edits(const Sequence& s, std::uint64_t budget = 0);

}  // namespace labsolve
