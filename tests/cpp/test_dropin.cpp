// Drop-in check of the C++ interface: same calls a user of the CPU reference would write
// (namespace skinnyqr, DenseMatrix / PanelPlan / exceptions), executed on the GPU through the C ABI.
// Prints a small JSON document that tests/test_cpp_dropin.py compares against the CPU oracle.
#include <cstdint>
#include <cstdio>
#include <string>
#include <vector>

#include "skinnyqr/gram_qr.hpp"
#include "skinnyqr/lstsq.hpp"
#include "skinnyqr/tsqr.hpp"

using namespace skinnyqr;

static std::uint64_t mix64(std::uint64_t seed, std::uint64_t index) {
  std::uint64_t z = seed + (index + 1u) * 0x9E3779B97F4A7C15ull;
  z ^= z >> 30; z *= 0xBF58476D1CE4E5B9ull;
  z ^= z >> 27; z *= 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

static DenseMatrix uniform_pm1(std::size_t m, std::size_t n, std::uint64_t seed) {
  DenseMatrix x(m, n);
  for (std::size_t e = 0; e < m * n; ++e)
    x.data()[e] = 2.0 * (static_cast<double>(mix64(seed, e) >> 11) * 0x1.0p-53) - 1.0;
  return x;
}

template <class M>
static void dump(const char* name, const M& a, std::size_t rows, std::size_t cols) {
  std::printf("\"%s\": [", name);
  for (std::size_t i = 0; i < rows * cols; ++i) std::printf("%s%.17g", i ? "," : "", a.data()[i]);
  std::printf("],\n");
}

int main() {
  const std::size_t m = 3001, n = 7;
  DenseMatrix x = uniform_pm1(m, n, 11);
  std::printf("{\n");
  UpperTriangular r = tsqr_qless(x, default_tsqr_plan(m, n));
  dump("tsqr_qless", r, n, n);
  UpperTriangular r2 = tsqr_qless(x, PanelPlan{5, 32, true});
  dump("tsqr_qless_k5_b32", r2, n, n);
  UpperTriangular rc = cholqr2(x, default_gram_plan(m, n));
  dump("cholqr2", rc, n, n);
  GramMatrix g = tsmttsm(x, default_gram_plan(m, n));
  dump("tsmttsm", g, n, n);
  QzResult qz = svqb2(x, default_gram_plan(m, n));
  dump("svqb2_sigma", qz.singular_values, n, 1);
  std::printf("\"svqb2_rank\": %zu,\n", qz.rank);
  std::vector<double> rhs(m);
  for (std::size_t i = 0; i < m; ++i) {
    rhs[i] = 0.25 * (static_cast<double>(mix64(12, i) >> 11) * 0x1.0p-53);
    for (std::size_t j = 0; j < n; ++j) rhs[i] += (j + 1.0) * x(i, j);
  }
  LstsqResult ls = solve_lstsq(x, rhs, LstsqMethod::tsqr);
  dump("lstsq_x", ls.x, n, 1);
  std::printf("\"lstsq_residual\": %.17g,\n", ls.residual_norm);
  std::string caught;
  try {
    GramMatrix bad(2);
    bad(0, 0) = bad(0, 1) = bad(1, 0) = bad(1, 1) = 1.0;
    cholesky(bad);
  } catch (const BreakdownError& e) {
    caught += "breakdown@" + std::to_string(e.pivot_index) + ";";
  }
  try {
    tsqr_qless(DenseMatrix(70, 65), PanelPlan{1, 130, true});
  } catch (const ArgumentError&) {
    caught += "argument;";
  }
  try {
    tsqr_qless(DenseMatrix(1, 3), PanelPlan{1, 8, true});
  } catch (const DimensionError&) {
    caught += "dimension;";
  }
  try {
    DenseMatrix z(50, 3);
    svqb2(z, PanelPlan{1, 16, true});
  } catch (const ZeroMatrixError&) {
    caught += "zero;";
  }
  std::printf("\"caught\": \"%s\"\n}\n", caught.c_str());
  return 0;
}
