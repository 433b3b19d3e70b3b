// Drop-in io.hpp against a file written by the unmodified reference (tests/golden/reference_5x3.tskm) and
// a write/read round trip; needs no CUDA library.
#include <cstdio>
#include "skinnyqr/io.hpp"
using namespace skinnyqr;
int main(int argc, char** argv) {
  DenseMatrix x = matrix_read(argv[1]);
  if (x.rows() != 5 || x.cols() != 3) return 2;
  for (std::size_t j = 0; j < 3; ++j)
    for (std::size_t i = 0; i < 5; ++i)
      if (x(i, j) != 0.5 * static_cast<double>(i) - 1.25 * static_cast<double>(j) + 1.0 / 3.0) return 3;
  matrix_write(argv[2], x);
  DenseMatrix y = matrix_read(argv[2]);
  for (std::size_t k = 0; k < 15; ++k)
    if (y.data()[k] != x.data()[k]) return 4;
  try { matrix_read(std::string(argv[2]) + ".missing"); return 5; } catch (const IoError&) {}
  std::puts("ok");
  return 0;
}
