// device.hpp — process-wide B200 context for the labsolve:: drop-in and the
// mapping from C-ABI status codes back to the reference's exception classes
// (invalid_argument / out_of_range / runtime_error).
#pragma once

#include <algorithm>
#include <stdexcept>
#include <string>
#include <vector>

#include "labs_b200.h"
#include "labsolve/memetic.hpp"

namespace labsolve::detail {

// Device 0 unless LABS_DEVICE says otherwise; created on first use. Throws
// std::runtime_error when no sm_100a device is present: there is no CPU path.
labs_ctx* device();

// The GPUs run_replicas spreads its replicas over: LABS_DEVICES (comma list,
// e.g. "0,1,2,3,4,5,6,7"; a device may repeat) or else {device()}.
const std::vector<labs_ctx*>& devices();

inline void check(int rc) {
  if (rc == LABS_OK) return;
  std::string msg = labs_last_error();
  switch (rc) {
    case LABS_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case LABS_ERR_OUT_OF_RANGE: throw std::out_of_range(msg);
    default: throw std::runtime_error(msg);
  }
}

// MemeticParams -> the C ABI's POD form. Optional budgets keep the
// reference's meaning for every value: a negative max_iterations or
// max_seconds stops at the first loop check (memetic.cpp:83-85 compares
// `iterations >= max` / `elapsed >= max`), i.e. it behaves as 0; only an
// absent optional is unlimited (the ABI's -1 sentinel).
inline labs_memetic_params device_params(int n, const MemeticParams& m) {
  if (n < 2) throw std::invalid_argument("memetic needs length >= 2");
  if (m.scan_workers < 1) throw std::invalid_argument("scan workers must be >= 1");
  if (m.p_mutate && !(*m.p_mutate > 0.0))
    throw std::invalid_argument("mutation probability must be in (0, 1]");
  labs_memetic_params p{};
  p.population_size = m.population_size;
  p.rng_kind = LABS_RNG_MT19937_64;
  p.p_comb = m.p_comb;
  p.p_mutate = m.p_mutate.value_or(-1.0);
  p.target_energy = m.target_energy;
  p.max_seconds = m.max_seconds ? std::max(0.0, *m.max_seconds) : -1.0;
  p.max_iterations = m.max_iterations ? std::max<long long>(0, *m.max_iterations) : -1;
  p.tabu = {m.tabu.min_tabu_factor, m.tabu.max_tabu_factor, LABS_TIE_REFERENCE, 0};
  return p;
}

// Memetic trace capacity per replica: max_iterations + 1 records when the
// run is bounded (every loop-top record fits), else `unbounded`.
inline int64_t trace_capacity(const MemeticParams& m, int64_t unbounded) {
  return m.max_iterations ? std::max<long long>(0, *m.max_iterations) + 1 : unbounded;
}

// The device reports how many records a replica produced; never truncate
// silently (the reference's MemeticTrace keeps every record).
inline void check_trace_len(int64_t len, int64_t cap) {
  if (len > cap)
    throw std::runtime_error("memetic trace exceeded its " + std::to_string(cap) +
                             "-record capacity; bound the run with max_iterations");
}

}  // namespace labsolve::detail
