#include "device.hpp"

#include <cstdlib>
#include <mutex>
#include <sstream>

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

const std::vector<labs_ctx*>& devices() {
  static std::once_flag once;
  static std::vector<labs_ctx*> ctxs;
  static int rc = LABS_OK;
  static std::string err;
  std::call_once(once, [] {
    const char* env = std::getenv("LABS_DEVICES");
    if (!env || !*env) return;
    std::stringstream ss(env);
    std::string tok;
    while (std::getline(ss, tok, ',')) {
      labs_ctx* c = nullptr;
      rc = labs_ctx_create(std::atoi(tok.c_str()), &c);
      if (rc != LABS_OK) {
        err = labs_last_error();
        return;
      }
      ctxs.push_back(c);
    }
  });
  if (rc != LABS_OK) throw std::runtime_error("B200 contexts (LABS_DEVICES): " + err);
  if (ctxs.empty()) {
    static std::vector<labs_ctx*> one;
    if (one.empty()) one.push_back(device());
    return one;
  }
  return ctxs;
}

}  // namespace labsolve::detail
