// runtime.cpp -- per-thread context + status mapping for the C++ drop-in
// (dropin/include/tq/b200_runtime.hpp).
#include "tq/b200_runtime.hpp"

#include <cstdlib>
#include <stdexcept>

namespace tq::b200 {

namespace {
struct ThreadContext {
  crys_ctx* ctx = nullptr;
  ~ThreadContext() {
    if (ctx) crys_destroy(ctx);
  }
};
}  // namespace

crys_ctx* context() {
  thread_local ThreadContext tc;
  if (!tc.ctx) {
    const char* e = std::getenv("CRYS_DEVICE");
    check(crys_init(e ? std::atoi(e) : 0, &tc.ctx));
  }
  return tc.ctx;
}

void raise(crys_status s) {
  const std::string msg = crys_last_error();
  switch (s) {
    case CRYS_ECONFIG: throw ConfigError(msg);
    case CRYS_ECONTRACT: throw ContractError(msg);
    case CRYS_EBUILD: throw BuildError(msg);
    case CRYS_EIO: throw IoError(msg);
    default: throw std::runtime_error("crystal_b200: " + msg);
  }
}

}  // namespace tq::b200
