// device.hpp — process-wide B200 context for the labsolve:: drop-in and the
// mapping from C-ABI status codes back to the reference's exception classes
// (invalid_argument / out_of_range / runtime_error).
#pragma once

#include <stdexcept>
#include <string>

#include "labs_b200.h"

namespace labsolve::detail {

// Device 0 unless LABS_DEVICE says otherwise; created on first use. Throws
// std::runtime_error when no sm_100a device is present: there is no CPU path.
labs_ctx* device();

inline void check(int rc) {
  if (rc == LABS_OK) return;
  std::string msg = labs_last_error();
  switch (rc) {
    case LABS_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case LABS_ERR_OUT_OF_RANGE: throw std::out_of_range(msg);
    default: throw std::runtime_error(msg);
  }
}

}  // namespace labsolve::detail
