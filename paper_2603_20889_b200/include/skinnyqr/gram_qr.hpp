// skinnyqr-b200: n x n factorisations and the Gram-based drivers
// (reference include/skinnyqr/gram_qr.hpp:13-59).  Everything between the two streaming passes of
// cholqr2 / svqb2 runs on the device.
#pragma once

#include <vector>

#include "skinnyqr/gram.hpp"
#include "skinnyqr/plan.hpp"
#include "skinnyqr/types.hpp"

namespace skinnyqr {

struct EigenDecomp {
  std::size_t order = 0;
  std::vector<double> values;  // descending
  DenseMatrix vectors;         // n x n orthogonal
};

struct QzResult {
  DenseMatrix transform;  // B
  DenseMatrix z;
  std::vector<double> singular_values;
  std::size_t rank = 0;
};

struct SvqbPassResult {
  DenseMatrix b;
  DenseMatrix z;
  std::vector<double> sigma;
  std::size_t rank = 0;
};

inline UpperTriangular cholesky(const GramMatrix& g) {
  UpperTriangular r(g.order());
  auto& c = b200::context();
  c.check(sqb_cholesky_host(c.get(), g.data(), g.order(), r.data()), "cholesky");
  return r;
}

inline EigenDecomp eigh_small(const GramMatrix& g) {
  EigenDecomp out;
  out.order = g.order();
  out.values.assign(g.order(), 0.0);
  out.vectors = DenseMatrix(g.order(), g.order());
  auto& c = b200::context();
  c.check(sqb_eigh_small_host(c.get(), g.data(), g.order(), out.values.data(), out.vectors.data()),
          "eigh_small");
  return out;
}

inline UpperTriangular cholqr2(const DenseMatrix& x, const PanelPlan& plan) {
  plan.validate();
  UpperTriangular r(x.cols());
  auto& c = b200::context();
  c.check(sqb_cholqr2_host(c.get(), x.data(), x.rows(), x.cols(), x.rows(), plan.num_blocks, plan.panel_rows,
                           r.data()),
          "cholqr2");
  return r;
}

inline SvqbPassResult svqb_pass(const DenseMatrix& x, const GramMatrix& g) {
  if (g.order() != x.cols()) throw DimensionError("svqb_pass: Gram order != cols of X");
  SvqbPassResult out;
  const std::size_t n = g.order();
  out.b = DenseMatrix(n, n);
  out.z = DenseMatrix(n, n);
  out.sigma.assign(n, 0.0);
  std::int64_t rank = 0;
  auto& c = b200::context();
  c.check(sqb_svqb_pass_host(c.get(), g.data(), n, out.b.data(), out.z.data(), out.sigma.data(), &rank),
          "svqb_pass");
  out.rank = static_cast<std::size_t>(rank);
  return out;
}

inline QzResult svqb2(const DenseMatrix& x, const PanelPlan& plan) {
  plan.validate();
  QzResult out;
  const std::size_t n = x.cols();
  out.transform = DenseMatrix(n, n);
  out.z = DenseMatrix(n, n);
  out.singular_values.assign(n, 0.0);
  std::int64_t rank = 0;
  auto& c = b200::context();
  c.check(sqb_svqb2_host(c.get(), x.data(), x.rows(), n, x.rows(), plan.num_blocks, plan.panel_rows,
                         out.transform.data(), out.z.data(), out.singular_values.data(), &rank),
          "svqb2");
  out.rank = static_cast<std::size_t>(rank);
  return out;
}

inline DenseMatrix reconstruct_q(const DenseMatrix& x, const UpperTriangular& r) {
  if (r.order() != x.cols()) throw DimensionError("reconstruct_q: R order != cols of X");
  DenseMatrix q(x.rows(), x.cols());
  auto& c = b200::context();
  c.check(sqb_reconstruct_q_host(c.get(), x.data(), x.rows(), x.cols(), x.rows(), r.data(), q.data(), x.rows()),
          "reconstruct_q");
  return q;
}

}  // namespace skinnyqr
