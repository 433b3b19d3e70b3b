// skinnyqr-b200: glue between the drop-in C++ interface and the C ABI (include/skinnyqr_b200.h).
#pragma once

#include <cstdint>
#include <string>

#include "skinnyqr/types.hpp"
#include "skinnyqr_b200.h"

namespace skinnyqr {
namespace b200 {

// Translates a C-ABI status into the reference's exception type (types.hpp error hierarchy).
[[noreturn]] inline void throw_status(int status, long long index, const char* where) {
  const std::string msg = std::string(where) + ": " + sqb_status_string(status);
  const std::size_t ix = index < 0 ? 0 : static_cast<std::size_t>(index);
  switch (status) {
    case SQB_E_DIMENSION: throw DimensionError(msg);
    case SQB_E_ARGUMENT: throw ArgumentError(msg);
    case SQB_E_BREAKDOWN: throw BreakdownError(msg, ix);
    case SQB_E_SINGULAR: throw SingularFactorError(msg, ix);
    case SQB_E_ZERO_MATRIX: throw ZeroMatrixError(msg);
    case SQB_E_RANK_DEFICIENT: throw RankDeficiencyError(msg, ix);
    default: throw Error(msg);
  }
}

// One context per thread (stream, workspaces, device status word); created on first use on the
// current CUDA device 0.  There is no CPU fallback: without an sm_100 device this throws.
class Context {
 public:
  explicit Context(int device = 0) {
    const int st = sqb_create(&ctx_, device);
    if (st != SQB_OK) throw_status(st, -1, "sqb_create");
  }
  ~Context() { sqb_destroy(ctx_); }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  sqb_context* get() const { return ctx_; }
  void check(int status, const char* where) const {
    if (status != SQB_OK) throw_status(status, sqb_last_error_index(ctx_), where);
  }

 private:
  sqb_context* ctx_ = nullptr;
};

inline Context& context() {
  thread_local Context ctx(0);
  return ctx;
}

}  // namespace b200
}  // namespace skinnyqr
