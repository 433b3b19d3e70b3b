// skinnyqr-b200: host-side value types and error classes of the drop-in C++ interface.
//
// Mirrors the public surface of the reference's include/skinnyqr/types.hpp (class names, members,
// accessors, column-major layout data[j*rows + i], error hierarchy :11-77, matrices :80-160,
// helpers :162-170) so that code written against the CPU reference compiles unchanged; the
// implementation is this project's own (one storage template, three thin aliases).
#pragma once

#include <cmath>
#include <cstddef>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace skinnyqr {

struct Error : std::runtime_error {
  using std::runtime_error::runtime_error;
};
#define SKINNYQR_B200_PLAIN_ERROR(Name, Base) \
  struct Name : Base {                        \
    using Base::Base;                         \
  }
SKINNYQR_B200_PLAIN_ERROR(IoError, Error);
SKINNYQR_B200_PLAIN_ERROR(FormatError, Error);
SKINNYQR_B200_PLAIN_ERROR(TruncationError, Error);
SKINNYQR_B200_PLAIN_ERROR(DimensionError, Error);
SKINNYQR_B200_PLAIN_ERROR(SizeOverflowError, Error);
SKINNYQR_B200_PLAIN_ERROR(ArgumentError, Error);
SKINNYQR_B200_PLAIN_ERROR(ZeroMatrixError, Error);
#undef SKINNYQR_B200_PLAIN_ERROR

struct BreakdownError : Error {
  BreakdownError(const std::string& what, std::size_t index) : Error(what), pivot_index(index) {}
  std::size_t pivot_index;
};
struct SingularFactorError : Error {
  SingularFactorError(const std::string& what, std::size_t index) : Error(what), diagonal_index(index) {}
  std::size_t diagonal_index;
};
struct RankDeficiencyError : Error {
  RankDeficiencyError(const std::string& what, std::size_t index) : Error(what), diagonal_index(index) {}
  std::size_t diagonal_index;
};

namespace detail {
// Column-major FP64 storage shared by the three matrix classes.
class ColumnStore {
 public:
  ColumnStore() = default;
  ColumnStore(std::size_t r, std::size_t c) : r_(r), c_(c), v_(r * c, 0.0) {}
  ColumnStore(std::size_t r, std::size_t c, std::vector<double> v) : r_(r), c_(c), v_(std::move(v)) {}
  std::size_t nrows() const { return r_; }
  std::size_t ncols() const { return c_; }
  double& at(std::size_t i, std::size_t j) { return v_[j * r_ + i]; }
  double at(std::size_t i, std::size_t j) const { return v_[j * r_ + i]; }
  double* raw() { return v_.data(); }
  const double* raw() const { return v_.data(); }
  std::size_t count() const { return v_.size(); }

 private:
  std::size_t r_ = 0, c_ = 0;
  std::vector<double> v_;
};
}  // namespace detail

// m x n dense matrix, element (i,j) at data()[j*rows() + i].
class DenseMatrix {
 public:
  DenseMatrix() = default;
  DenseMatrix(std::size_t rows, std::size_t cols) : s_(rows, cols) {}
  DenseMatrix(std::size_t rows, std::size_t cols, std::vector<double> data)
      : s_(rows, cols, std::move(data)) {
    if (s_.count() != rows * cols) throw DimensionError("DenseMatrix: data length != rows*cols");
  }
  std::size_t rows() const { return s_.nrows(); }
  std::size_t cols() const { return s_.ncols(); }
  double& operator()(std::size_t i, std::size_t j) { return s_.at(i, j); }
  double operator()(std::size_t i, std::size_t j) const { return s_.at(i, j); }
  double* col(std::size_t j) { return s_.raw() + j * rows(); }
  const double* col(std::size_t j) const { return s_.raw() + j * rows(); }
  double* data() { return s_.raw(); }
  const double* data() const { return s_.raw(); }
  const std::string& label() const { return label_; }
  void set_label(std::string l) { label_ = std::move(l); }

 private:
  detail::ColumnStore s_;
  std::string label_;
};

// n x n upper triangular factor stored as a full square; strict lower part exactly zero.
class UpperTriangular {
 public:
  UpperTriangular() = default;
  explicit UpperTriangular(std::size_t order) : s_(order, order) {}
  std::size_t order() const { return s_.nrows(); }
  double& operator()(std::size_t i, std::size_t j) { return s_.at(i, j); }
  double operator()(std::size_t i, std::size_t j) const { return s_.at(i, j); }
  double* data() { return s_.raw(); }
  const double* data() const { return s_.raw(); }

 private:
  detail::ColumnStore s_;
};

// Symmetric n x n Gram matrix, full storage.
class GramMatrix {
 public:
  GramMatrix() = default;
  explicit GramMatrix(std::size_t order) : s_(order, order) {}
  std::size_t order() const { return s_.nrows(); }
  double& operator()(std::size_t i, std::size_t j) { return s_.at(i, j); }
  double operator()(std::size_t i, std::size_t j) const { return s_.at(i, j); }
  double* data() { return s_.raw(); }
  const double* data() const { return s_.raw(); }
  void mirror_upper() {
    const std::size_t n = order();
    for (std::size_t c = 1; c < n; ++c)
      for (std::size_t r = 0; r < c; ++r) s_.at(c, r) = s_.at(r, c);
  }

 private:
  detail::ColumnStore s_;
};

// Row i of R is negated from the diagonal on whenever R(i,i) < 0 (reference types.cpp:8-14).
inline void sign_normalize(UpperTriangular& r) {
  const std::size_t n = r.order();
  for (std::size_t i = 0; i < n; ++i) {
    if (!(r(i, i) < 0.0)) continue;
    for (std::size_t j = i; j < n; ++j) r(i, j) = -r(i, j);
  }
}

// Frobenius norm, pairwise over blocks of 256 (reference types.cpp:16-38).
inline double frobenius_norm(const DenseMatrix& x) {
  const std::size_t total = x.rows() * x.cols();
  const double* p = x.data();
  std::vector<double> level;
  for (std::size_t off = 0; off < total; off += 256) {
    double s = 0.0;
    const std::size_t stop = off + 256 < total ? off + 256 : total;
    for (std::size_t t = off; t < stop; ++t) s += p[t] * p[t];
    level.push_back(s);
  }
  while (level.size() > 1) {
    std::vector<double> next;
    for (std::size_t t = 0; t + 1 < level.size(); t += 2) next.push_back(level[t] + level[t + 1]);
    if (level.size() % 2) next.push_back(level.back());
    level.swap(next);
  }
  return level.empty() ? 0.0 : std::sqrt(level[0]);
}

// rows >= cols >= 1 and all entries finite, else DimensionError / ArgumentError
// (reference types.cpp:40-48).  The GPU entry points do NOT call this host scan: they fuse the
// finiteness test into the streaming kernels and raise the same ArgumentError afterwards.
inline void validate_factorization_input(const DenseMatrix& x, const char* op) {
  if (x.cols() < 1 || x.rows() < x.cols())
    throw DimensionError(std::string(op) + ": need rows >= cols >= 1");
  const std::size_t total = x.rows() * x.cols();
  for (std::size_t t = 0; t < total; ++t)
    if (!std::isfinite(x.data()[t])) throw ArgumentError(std::string(op) + ": non-finite entry");
}

}  // namespace skinnyqr
