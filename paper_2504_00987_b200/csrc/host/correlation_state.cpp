// labsolve::CorrelationState and scan_neighborhood on the B200 engine.
#include "labsolve/correlation_state.hpp"

#include <stdexcept>

#include "device.hpp"

namespace labsolve {

CorrelationState::CorrelationState(const Sequence& s) : n_(s.size()), pivot_(s) {
  if (n_ < 2) throw std::invalid_argument("correlation state needs length >= 2");
  labs_eval* e = nullptr;
  detail::check(labs_eval_create(detail::device(), n_, &e));
  eval_ = std::shared_ptr<labs_eval>(e, labs_eval_destroy);
  evaluate();
}

// One device pass: C_k, E and every neighbor energy of the pivot.
void CorrelationState::evaluate() {
  corr_.assign(n_ - 1, 0);
  neighbors_.assign(n_, 0);
  int64_t e = 0;
  detail::check(labs_eval_run(eval_.get(), pivot_.data(), corr_.data(), &e,
                              reinterpret_cast<int64_t*>(neighbors_.data())));
  energy_ = e;
}

long long CorrelationState::correlation(int k) const {
  if (k < 1 || k >= n_) throw std::out_of_range("correlation lag");
  return corr_[k - 1];
}

int CorrelationState::product(int k, int i) const {
  if (k < 1 || k >= n_) throw std::out_of_range("product lag");
  if (i < 0 || i + k >= n_) throw std::out_of_range("product index");
  return pivot_.spin(i) * pivot_.spin(i + k);
}

std::size_t CorrelationState::table_bytes() const {
  const std::size_t pairs = static_cast<std::size_t>(n_) * (n_ - 1) / 2;
  return (pairs + 7) / 8;
}

long long CorrelationState::neighbor_energy(int j, std::uint64_t* touches) const {
  if (j < 0 || j >= n_) throw std::out_of_range("flip position");
  if (touches) *touches += static_cast<std::uint64_t>(n_ - 1);
  return neighbors_[j];
}

void CorrelationState::apply_flip(int j, std::uint64_t* touches) {
  if (j < 0 || j >= n_) throw std::out_of_range("flip position");
  if (touches) *touches += static_cast<std::uint64_t>(n_ - 1);
  pivot_.flip(j);
  evaluate();
}

ScanResult scan_neighborhood(const CorrelationState& state,
                             const std::function<bool(int)>& admissible, Rng& rng,
                             int workers, bool allow_fallback) {
  if (workers < 1) throw std::invalid_argument("scan workers must be >= 1");
  const int n = state.size();
  std::vector<uint8_t> mask(n);
  for (int j = 0; j < n; ++j) mask[j] = admissible(j) ? 1 : 0;
  int32_t pos = -1, fb = 0, ntie = 0;
  int64_t e = 0;
  const int rc = labs_scan(detail::device(), n, 1, state.pivot().data(), mask.data(),
                           &rng.state(), allow_fallback ? 1 : 0, LABS_TIE_REFERENCE, &pos, &e,
                           &fb, &ntie, nullptr);
  if (rc == LABS_ERR_RUNTIME)
    throw std::runtime_error("no admissible position in neighborhood scan");
  detail::check(rc);
  return {pos, e, fb != 0};
}

}  // namespace labsolve
