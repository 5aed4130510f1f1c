// Probe of the skew.hpp drop-in (device deviation) for tests/test_skew_gpu.py:
// stdin lines "n budget edits w0 [w1 ...]" -> "value exceeded evaluations".
#include <cstdint>
#include <iostream>
#include <sstream>
#include <string>

#include "labsolve/skew.hpp"

int main() {
  std::string line;
  while (std::getline(std::cin, line)) {
    std::istringstream in(line);
    int n, edits;
    unsigned long long budget;
    in >> n >> budget >> edits;
    labsolve::Sequence s(n);
    unsigned long long w;
    for (int i = 0; i < s.word_count() && (in >> w); ++i) s.set_word(i, w);
    const labsolve::DeviationResult d = edits ? labsolve::deviation_with_edits(s, budget)
                                              : labsolve::deviation(s, budget);
    std::cout << d.value << ' ' << (d.budget_exceeded ? 1 : 0) << ' ' << d.evaluations << '\n';
  }
  return 0;
}
