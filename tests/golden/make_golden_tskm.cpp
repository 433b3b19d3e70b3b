#include "skinnyqr/io.hpp"
using namespace skinnyqr;
int main(int argc, char** argv) {
  DenseMatrix x(5, 3);
  for (std::size_t j = 0; j < 3; ++j)
    for (std::size_t i = 0; i < 5; ++i) x(i, j) = 0.5 * static_cast<double>(i) - 1.25 * static_cast<double>(j) + 1.0 / 3.0;
  matrix_write(argv[1], x);
  DenseMatrix y = matrix_read(argv[2]);
  return (y.rows() == 4 && y.cols() == 2 && y(3, 1) == 7.0) ? 0 : 3;
}
