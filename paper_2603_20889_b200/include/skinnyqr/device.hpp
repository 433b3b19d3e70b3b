// skinnyqr-b200: device-resident operands for C++ callers.
//
// The drop-in entry points (tsqr.hpp, gram.hpp, gram_qr.hpp, lstsq.hpp) take the reference's host types and
// pay for the PCIe transfer of X on every call.  Production code keeps X in HBM: DeviceMatrix owns a
// column-major FP64 matrix on the GPU (allocated and filled through the C ABI, so the caller needs no CUDA
// headers), and the overloads below run the same methods on it - only the n x n results come back to the
// host.  The row-sharded variants are the multi-GPU form: one process per GPU, every rank passes its own
// row slab, all ranks receive the same result (NCCL inside the library, or a transport installed with
// sqb_set_allgather).  Reference interfaces: include/skinnyqr/tsqr.hpp:59-68, gram.hpp:12-21,
// gram_qr.hpp:37-59, lstsq.hpp:21.
#pragma once

#include <array>
#include <cstdint>
#include <utility>
#include <vector>

#include "skinnyqr/gram_qr.hpp"
#include "skinnyqr/lstsq.hpp"
#include "skinnyqr/tsqr.hpp"

namespace skinnyqr {
namespace b200 {

class DeviceMatrix {
 public:
  DeviceMatrix() = default;
  DeviceMatrix(std::size_t rows, std::size_t cols) : rows_(rows), cols_(cols) {
    auto& c = context();
    c.check(sqb_device_alloc(c.get(), static_cast<std::int64_t>(sizeof(double) * rows * cols), &ptr_), "DeviceMatrix");
  }
  explicit DeviceMatrix(const DenseMatrix& host) : DeviceMatrix(host.rows(), host.cols()) {
    auto& c = context();
    c.check(sqb_copy_h2d(c.get(), ptr_, host.data(), static_cast<std::int64_t>(sizeof(double) * rows_ * cols_)),
            "DeviceMatrix(host)");
  }
  DeviceMatrix(const DeviceMatrix&) = delete;
  DeviceMatrix& operator=(const DeviceMatrix&) = delete;
  DeviceMatrix(DeviceMatrix&& o) noexcept { swap(o); }
  DeviceMatrix& operator=(DeviceMatrix&& o) noexcept {
    swap(o);
    return *this;
  }
  ~DeviceMatrix() {
    if (ptr_) sqb_device_free(context().get(), ptr_);
  }
  // synthetic input generated in place (reference generator streams, src/matgen.cpp:8-17): rows
  // [row_offset, row_offset + rows) of a logical m_total x cols Gaussian matrix
  void fill_gaussian(std::uint64_t seed, std::size_t row_offset = 0, std::size_t m_total = 0) {
    auto& c = context();
    c.check(sqb_fill_gaussian_dev(c.get(), data(), rows_, cols_, rows_, seed, row_offset, m_total ? m_total : rows_),
            "fill_gaussian");
  }
  DenseMatrix to_host() const {
    DenseMatrix h(rows_, cols_);
    auto& c = context();
    c.check(sqb_copy_d2h(c.get(), h.data(), ptr_, static_cast<std::int64_t>(sizeof(double) * rows_ * cols_)), "to_host");
    return h;
  }
  double* data() { return static_cast<double*>(ptr_); }
  const double* data() const { return static_cast<const double*>(ptr_); }
  std::size_t rows() const { return rows_; }
  std::size_t cols() const { return cols_; }
  std::size_t ld() const { return rows_; }

 private:
  void swap(DeviceMatrix& o) {
    std::swap(ptr_, o.ptr_);
    std::swap(rows_, o.rows_);
    std::swap(cols_, o.cols_);
  }
  void* ptr_ = nullptr;
  std::size_t rows_ = 0, cols_ = 0;
};

namespace detail {
// n x n (or shorter) result: device scratch -> host object, then the device status of the whole call
template <class Host>
inline void fetch(const DeviceMatrix& d, Host& h, std::size_t count, const char* where) {
  auto& c = context();
  c.check(sqb_copy_d2h(c.get(), h.data(), d.data(), static_cast<std::int64_t>(sizeof(double) * count)), where);
}
inline void finish(const char* where) {
  auto& c = context();
  c.check(sqb_sync(c.get()), where);
}
}  // namespace detail

// PanelPlan{0, 0}: the device default (one CTA per SM, kernel panel height)
inline UpperTriangular tsqr_qless(const DeviceMatrix& x, std::size_t num_blocks = 0, std::size_t panel_rows = 0) {
  const std::size_t n = x.cols();
  DeviceMatrix dr(n, n);
  UpperTriangular r(n);
  auto& c = context();
  c.check(sqb_tsqr_qless_dev(c.get(), x.data(), x.rows(), n, x.ld(), num_blocks, panel_rows, dr.data()), "tsqr_qless");
  detail::fetch(dr, r, n * n, "tsqr_qless");
  detail::finish("tsqr_qless");
  return r;
}

inline GramMatrix tsmttsm(const DeviceMatrix& x, std::size_t num_blocks = 0, std::size_t panel_rows = 0) {
  const std::size_t n = x.cols();
  DeviceMatrix dc(n, n);
  GramMatrix g(n);
  auto& c = context();
  c.check(sqb_tsmttsm_dev(c.get(), x.data(), x.rows(), n, x.ld(), num_blocks, panel_rows, dc.data()), "tsmttsm");
  detail::fetch(dc, g, n * n, "tsmttsm");
  detail::finish("tsmttsm");
  return g;
}

inline UpperTriangular cholqr2(const DeviceMatrix& x, std::size_t num_blocks = 0, std::size_t panel_rows = 0) {
  const std::size_t n = x.cols();
  DeviceMatrix dr(n, n);
  UpperTriangular r(n);
  auto& c = context();
  c.check(sqb_cholqr2_dev(c.get(), x.data(), x.rows(), n, x.ld(), num_blocks, panel_rows, dr.data()), "cholqr2");
  detail::fetch(dr, r, n * n, "cholqr2");
  detail::finish("cholqr2");
  return r;
}

inline QzResult svqb2(const DeviceMatrix& x, std::size_t num_blocks = 0, std::size_t panel_rows = 0) {
  const std::size_t n = x.cols();
  DeviceMatrix dt(n, n), dz(n, n), ds(n + 1, 1);  // sigma (n) and the rank word
  QzResult out;
  out.transform = DenseMatrix(n, n);
  out.z = DenseMatrix(n, n);
  out.singular_values.assign(n, 0.0);
  auto& c = context();
  std::int64_t* d_rank = reinterpret_cast<std::int64_t*>(ds.data() + n);
  c.check(sqb_svqb2_dev(c.get(), x.data(), x.rows(), n, x.ld(), num_blocks, panel_rows, dt.data(), dz.data(), ds.data(),
                        d_rank),
          "svqb2");
  detail::fetch(dt, out.transform, n * n, "svqb2");
  detail::fetch(dz, out.z, n * n, "svqb2");
  detail::fetch(ds, out.singular_values, n, "svqb2");
  std::int64_t rank = 0;
  c.check(sqb_copy_d2h(c.get(), &rank, d_rank, sizeof(rank)), "svqb2");
  detail::finish("svqb2");
  out.rank = static_cast<std::size_t>(rank);
  return out;
}

// A (m x n) and rhs (m x 1) stay separate device arrays; [A rhs] is never assembled (lstsq.cpp:24-26)
inline LstsqResult solve_lstsq(const DeviceMatrix& a, const DeviceMatrix& rhs, LstsqMethod method) {
  if (rhs.rows() != a.rows() || rhs.cols() != 1) throw DimensionError("solve_lstsq: rhs must be rows(A) x 1");
  const std::size_t n = a.cols();
  DeviceMatrix dx(n + 1, 1);
  LstsqResult out;
  out.x.assign(n, 0.0);
  const int meth = method == LstsqMethod::tsqr ? SQB_METHOD_TSQR
                   : method == LstsqMethod::cholqr2 ? SQB_METHOD_CHOLQR2 : SQB_METHOD_SVQB2;
  auto& c = context();
  c.check(sqb_solve_lstsq_dev(c.get(), a.data(), a.rows(), n, a.ld(), rhs.data(), meth, dx.data(), dx.data() + n),
          "solve_lstsq");
  detail::fetch(dx, out.x, n, "solve_lstsq");
  c.check(sqb_copy_d2h(c.get(), &out.residual_norm, dx.data() + n, sizeof(double)), "solve_lstsq");
  detail::finish("solve_lstsq");
  return out;
}

// ---- row-sharded (multi-GPU) forms: rank g passes its slab, every rank gets the same result -------------
inline std::array<char, 128> nccl_unique_id() {
  std::array<char, 128> id{};
  if (sqb_nccl_unique_id(id.data()) != SQB_OK) throw Error("nccl_unique_id: NCCL not available");
  return id;
}
inline void init_sharded(const std::array<char, 128>& id, int rank, int world) {
  auto& c = context();
  c.check(sqb_init_nccl(c.get(), id.data(), rank, world), "init_sharded");
}
inline void set_allgather(sqb_allgather_fn fn, void* user, int rank, int world) {
  auto& c = context();
  c.check(sqb_set_allgather(c.get(), fn, user, rank, world), "set_allgather");
}

inline UpperTriangular tsqr_qless_sharded(const DeviceMatrix& slab) {
  const std::size_t n = slab.cols();
  DeviceMatrix dr(n, n);
  UpperTriangular r(n);
  auto& c = context();
  c.check(sqb_tsqr_qless_sharded_dev(c.get(), slab.data(), slab.rows(), n, slab.ld(), dr.data()), "tsqr_qless_sharded");
  detail::fetch(dr, r, n * n, "tsqr_qless_sharded");
  detail::finish("tsqr_qless_sharded");
  return r;
}

inline UpperTriangular cholqr2_sharded(const DeviceMatrix& slab) {
  const std::size_t n = slab.cols();
  DeviceMatrix dr(n, n);
  UpperTriangular r(n);
  auto& c = context();
  c.check(sqb_cholqr2_sharded_dev(c.get(), slab.data(), slab.rows(), n, slab.ld(), dr.data()), "cholqr2_sharded");
  detail::fetch(dr, r, n * n, "cholqr2_sharded");
  detail::finish("cholqr2_sharded");
  return r;
}

inline LstsqResult solve_lstsq_sharded(const DeviceMatrix& a_slab, const DeviceMatrix& rhs_slab) {
  if (rhs_slab.rows() != a_slab.rows() || rhs_slab.cols() != 1)
    throw DimensionError("solve_lstsq_sharded: rhs must be rows(A) x 1");
  const std::size_t n = a_slab.cols();
  DeviceMatrix dx(n + 1, 1);
  LstsqResult out;
  out.x.assign(n, 0.0);
  auto& c = context();
  c.check(sqb_solve_lstsq_sharded_dev(c.get(), a_slab.data(), a_slab.rows(), n, a_slab.ld(), rhs_slab.data(), dx.data(),
                                      dx.data() + n),
          "solve_lstsq_sharded");
  detail::fetch(dx, out.x, n, "solve_lstsq_sharded");
  c.check(sqb_copy_d2h(c.get(), &out.residual_norm, dx.data() + n, sizeof(double)), "solve_lstsq_sharded");
  detail::finish("solve_lstsq_sharded");
  return out;
}

}  // namespace b200
}  // namespace skinnyqr
