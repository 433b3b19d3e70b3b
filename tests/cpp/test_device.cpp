// Device-resident C++ interface (paper_2603_20889_b200/include/skinnyqr/device.hpp): X lives in HBM, only the
// n x n results come back.  Also the row-sharded form with a caller-supplied all-gather: this process plays
// rank 0 of a 2-rank world, the callback serves rank 1's block, which was computed beforehand with
// sqb_tsqr_local_dev on the second row slab.  Prints JSON for tests/test_cpp_dropin.py.
#include <cstdint>
#include <cstdio>
#include <vector>

#include "skinnyqr/device.hpp"

using namespace skinnyqr;

static std::uint64_t mix64(std::uint64_t seed, std::uint64_t index) {
  std::uint64_t z = seed + (index + 1u) * 0x9E3779B97F4A7C15ull;
  z ^= z >> 30; z *= 0xBF58476D1CE4E5B9ull;
  z ^= z >> 27; z *= 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

template <class M>
static void dump(const char* name, const M& a, std::size_t count, bool last = false) {
  std::printf("\"%s\": [", name);
  for (std::size_t i = 0; i < count; ++i) std::printf("%s%.17g", i ? "," : "", a.data()[i]);
  std::printf("]%s\n", last ? "" : ",");
}

struct Exchange {
  const double* d_other;  // rank 1's n x n block (device)
  std::size_t count;
  int calls;
};

// all-gather for world = 2, rank = 0: recv = [own block | rank 1's block], staged through the host
static int serve_allgather(void* user, const double* d_send, double* d_recv, std::int64_t count) {
  auto* ex = static_cast<Exchange*>(user);
  if (static_cast<std::size_t>(count) != ex->count) return 1;
  std::vector<double> h(2 * count);
  sqb_context* c = b200::context().get();
  if (sqb_copy_d2h(c, h.data(), d_send, sizeof(double) * count) != SQB_OK) return 1;
  if (sqb_copy_d2h(c, h.data() + count, ex->d_other, sizeof(double) * count) != SQB_OK) return 1;
  ex->calls++;
  return sqb_copy_h2d(c, d_recv, h.data(), sizeof(double) * 2 * count) == SQB_OK ? 0 : 1;
}

int main() {
  const std::size_t m = 30011, n = 9, m0 = 15006;
  DenseMatrix x(m, n);
  for (std::size_t e = 0; e < m * n; ++e) x.data()[e] = 2.0 * (static_cast<double>(mix64(21, e) >> 11) * 0x1.0p-53) - 1.0;
  DenseMatrix rhs(m, 1);
  for (std::size_t i = 0; i < m; ++i) {
    rhs(i, 0) = 0.125 * (static_cast<double>(mix64(22, i) >> 11) * 0x1.0p-53);
    for (std::size_t j = 0; j < n; ++j) rhs(i, 0) += (j + 1.0) * x(i, j);
  }
  b200::DeviceMatrix dx(x), drhs(rhs);
  std::printf("{\n");
  dump("tsqr_qless", b200::tsqr_qless(dx), n * n);
  dump("tsqr_qless_k7_b64", b200::tsqr_qless(dx, 7, 64), n * n);
  dump("cholqr2", b200::cholqr2(dx), n * n);
  dump("tsmttsm", b200::tsmttsm(dx), n * n);
  QzResult qz = b200::svqb2(dx);
  dump("svqb2_sigma", qz.singular_values, n);
  std::printf("\"svqb2_rank\": %zu,\n", qz.rank);
  LstsqResult ls = b200::solve_lstsq(dx, drhs, LstsqMethod::tsqr);
  dump("lstsq_x", ls.x, n);
  std::printf("\"lstsq_residual\": %.17g,\n", ls.residual_norm);
  dump("roundtrip", dx.to_host(), 16);

  // two row slabs as their own allocations (what each rank of a sharded run holds)
  DenseMatrix s0(m0, n), s1(m - m0, n), b0(m0, 1), b1(m - m0, 1);
  for (std::size_t j = 0; j < n; ++j) {
    for (std::size_t i = 0; i < m0; ++i) s0(i, j) = x(i, j);
    for (std::size_t i = m0; i < m; ++i) s1(i - m0, j) = x(i, j);
  }
  for (std::size_t i = 0; i < m0; ++i) b0(i, 0) = rhs(i, 0);
  for (std::size_t i = m0; i < m; ++i) b1(i - m0, 0) = rhs(i, 0);
  b200::DeviceMatrix d0(s0), d1(s1), db0(b0), db1(b1);
  auto& c = b200::context();
  // rank 1's contributions, computed up front: its TSQR triangle of [A] and of [A rhs]
  b200::DeviceMatrix other(n, n), other_ls(n + 1, n + 1), a1b1(m - m0, n + 1);
  c.check(sqb_tsqr_local_dev(c.get(), d1.data(), d1.rows(), n, d1.ld(), other.data()), "tsqr_local");
  {
    DenseMatrix e(m - m0, n + 1);
    for (std::size_t j = 0; j < n; ++j)
      for (std::size_t i = 0; i < m - m0; ++i) e(i, j) = s1(i, j);
    for (std::size_t i = 0; i < m - m0; ++i) e(i, n) = b1(i, 0);
    b200::DeviceMatrix de(e);
    c.check(sqb_tsqr_local_dev(c.get(), de.data(), de.rows(), n + 1, de.ld(), other_ls.data()), "tsqr_local");
    c.check(sqb_sync(c.get()), "sync");
  }
  Exchange ex{other.data(), n * n, 0};
  b200::set_allgather(serve_allgather, &ex, 0, 2);
  dump("tsqr_qless_sharded", b200::tsqr_qless_sharded(d0), n * n);
  Exchange ex2{other_ls.data(), (n + 1) * (n + 1), 0};
  b200::set_allgather(serve_allgather, &ex2, 0, 2);
  LstsqResult lss = b200::solve_lstsq_sharded(d0, db0);
  dump("lstsq_sharded_x", lss.x, n);
  std::printf("\"lstsq_sharded_residual\": %.17g,\n", lss.residual_norm);
  std::printf("\"exchange_calls\": %d\n}\n", ex.calls + ex2.calls);
  return 0;
}
