// skinnyqr-b200: fused Gram kernels (reference include/skinnyqr/gram.hpp:12-24).
#pragma once

#include <cfloat>
#include <cmath>

#include "skinnyqr/plan.hpp"
#include "skinnyqr/types.hpp"

namespace skinnyqr {

inline GramMatrix tsmttsm(const DenseMatrix& x, const PanelPlan& plan) {
  plan.validate();
  GramMatrix g(x.cols());
  auto& c = b200::context();
  c.check(sqb_tsmttsm_host(c.get(), x.data(), x.rows(), x.cols(), x.rows(), plan.num_blocks, plan.panel_rows,
                           g.data()),
          "tsmttsm");
  return g;
}

inline GramMatrix tsmRttsmR(const DenseMatrix& x, const UpperTriangular& r, const PanelPlan& plan) {
  plan.validate();
  if (r.order() != x.cols()) throw DimensionError("tsmRttsmR: R order != cols of X");
  GramMatrix g(x.cols());
  auto& c = b200::context();
  c.check(sqb_tsmRttsmR_host(c.get(), x.data(), x.rows(), x.cols(), x.rows(), r.data(), plan.num_blocks,
                             plan.panel_rows, g.data()),
          "tsmRttsmR");
  return g;
}

inline GramMatrix tsmmttsmm(const DenseMatrix& x, const DenseMatrix& b, const PanelPlan& plan) {
  plan.validate();
  if (b.rows() != x.cols() || b.cols() != x.cols()) throw DimensionError("tsmmttsmm: B must be n x n");
  GramMatrix g(x.cols());
  auto& c = b200::context();
  c.check(sqb_tsmmttsmm_host(c.get(), x.data(), x.rows(), x.cols(), x.rows(), b.data(), plan.num_blocks,
                             plan.panel_rows, g.data()),
          "tsmmttsmm");
  return g;
}

// n * eps * max|diag(R)| (reference gram.cpp:106-111)
inline double trsm_diag_tolerance(const UpperTriangular& r) {
  double top = 0.0;
  for (std::size_t j = 0; j < r.order(); ++j) top = std::fmax(top, std::fabs(r(j, j)));
  return static_cast<double>(r.order()) * DBL_EPSILON * top;
}

}  // namespace skinnyqr
