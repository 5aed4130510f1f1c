#include "device.hpp"

#include <cstdlib>
#include <mutex>

namespace labsolve::detail {

labs_ctx* device() {
  static std::once_flag once;
  static labs_ctx* ctx = nullptr;
  static int rc = LABS_OK;
  static std::string err;
  std::call_once(once, [] {
    const char* env = std::getenv("LABS_DEVICE");
    rc = labs_ctx_create(env ? std::atoi(env) : 0, &ctx);
    if (rc != LABS_OK) err = labs_last_error();
  });
  if (rc != LABS_OK) throw std::runtime_error("B200 context: " + err);
  return ctx;
}

}  // namespace labsolve::detail
