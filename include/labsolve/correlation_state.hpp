// correlation_state.hpp — drop-in for
// /root/reference/proj/include/labsolve/correlation_state.hpp:17-63.
//
// The reference keeps a packed product table and answers neighbor_energy(j)
// with an O(n) walk over it. Here the state is evaluated on the B200: a build
// (or commit) runs the device engine once and caches C_k, E and all n
// neighbor energies, so neighbor_energy(j) is a lookup. Each object owns a
// persistent device evaluator (labs_eval: no allocation per commit; one
// H2D + launch + D2H). A commit is still a device round trip: callers that
// flip long known sequences should batch them with labs_flip_trace. `touches` keeps the
// reference's accounting (n-1 product entries per query or flip) so callers
// that budget work with it see the same numbers.
#pragma once

#include <cstddef>
#include <cstdint>
#include <functional>
#include <memory>
#include <vector>

#include "labsolve/rng.hpp"
#include "labsolve/sequence.hpp"

struct labs_eval;  // the device evaluator (include/labs_b200.h)

namespace labsolve {

class CorrelationState {
 public:
  explicit CorrelationState(const Sequence& s);

  int size() const { return n_; }
  const Sequence& pivot() const { return pivot_; }
  long long energy() const { return energy_; }

  long long correlation(int k) const;
  int product(int k, int i) const;
  // Size the reference's packed product table would occupy.
  std::size_t table_bytes() const;

  long long neighbor_energy(int j, std::uint64_t* touches = nullptr) const;
  void apply_flip(int j, std::uint64_t* touches = nullptr);

 private:
  void evaluate();

  int n_ = 0;
  Sequence pivot_;
  // device scratch shared by copies (every evaluation re-uploads the pivot;
  // the results live in the members below)
  std::shared_ptr<::labs_eval> eval_;
  std::vector<std::int32_t> corr_;
  std::vector<long long> neighbors_;
  long long energy_ = 0;
};

struct ScanResult {
  int position = -1;
  long long energy = 0;
  bool fallback = false;
};

// `workers` is accepted for compatibility: the device scan is one warp and is
// partition-independent by construction.
ScanResult scan_neighborhood(const CorrelationState& state,
                             const std::function<bool(int)>& admissible,
                             Rng& rng, int workers = 1,
                             bool allow_fallback = true);

}  // namespace labsolve
