// skinnyqr-b200: single-pass least squares via Q-less QR of [A rhs]
// (reference include/skinnyqr/lstsq.hpp:9-22).  A and rhs are uploaded as they are; the extended
// matrix of the reference (src/lstsq.cpp:24-26) is never assembled on the host.
#pragma once

#include <vector>

#include "skinnyqr/plan.hpp"
#include "skinnyqr/types.hpp"

namespace skinnyqr {

enum class LstsqMethod { tsqr, cholqr2, svqb2 };

struct LstsqResult {
  std::vector<double> x;
  double residual_norm = 0.0;
};

inline LstsqResult solve_lstsq(const DenseMatrix& a, const std::vector<double>& rhs, LstsqMethod method) {
  if (rhs.size() != a.rows()) throw DimensionError("solve_lstsq: rhs length != rows of A");
  LstsqResult out;
  out.x.assign(a.cols(), 0.0);
  const int meth = method == LstsqMethod::tsqr ? SQB_METHOD_TSQR
                   : method == LstsqMethod::cholqr2 ? SQB_METHOD_CHOLQR2 : SQB_METHOD_SVQB2;
  auto& c = b200::context();
  c.check(sqb_solve_lstsq_host(c.get(), a.data(), a.rows(), a.cols(), a.rows(), rhs.data(), meth, out.x.data(),
                               &out.residual_norm),
          "solve_lstsq");
  return out;
}

}  // namespace skinnyqr
