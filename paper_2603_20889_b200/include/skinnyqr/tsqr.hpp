// skinnyqr-b200: Q-less Householder TSQR entry points (reference include/skinnyqr/tsqr.hpp:59-68).
// TrapezoidalWorkspace / factor_trapezoidal / reference_hhqr are CPU internals of the reference
// and have no GPU counterpart (the CUDA kernels keep their panel in registers).
#pragma once

#include "skinnyqr/plan.hpp"
#include "skinnyqr/types.hpp"

namespace skinnyqr {

inline UpperTriangular block_qless_qr(const DenseMatrix& xi, std::size_t b) {
  UpperTriangular r(xi.cols());
  auto& c = b200::context();
  c.check(sqb_block_qless_qr_host(c.get(), xi.data(), xi.rows(), xi.cols(), xi.rows(), b, r.data()),
          "block_qless_qr");
  return r;
}

inline UpperTriangular tsqr_qless(const DenseMatrix& x, const PanelPlan& plan) {
  plan.validate();
  UpperTriangular r(x.cols());
  auto& c = b200::context();
  c.check(sqb_tsqr_qless_host(c.get(), x.data(), x.rows(), x.cols(), x.rows(), plan.num_blocks,
                              plan.panel_rows, r.data()),
          "tsqr_qless");
  return r;
}

inline DenseMatrix tsqr_stage1(const DenseMatrix& x, const PanelPlan& plan) {
  plan.validate();
  DenseMatrix y(plan.num_blocks * x.cols(), x.cols());
  auto& c = b200::context();
  c.check(sqb_tsqr_stage1_host(c.get(), x.data(), x.rows(), x.cols(), x.rows(), plan.num_blocks,
                               plan.panel_rows, y.data()),
          "tsqr_stage1");
  return y;
}

}  // namespace skinnyqr
