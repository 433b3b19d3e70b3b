// Compiles against the drop-in headers only (no CUDA library needed): the Roofline model mirror of the
// reference's include/skinnyqr/perf_model.hpp, checked against the SPEC examples.
#include <cassert>
#include <cmath>
#include <cstdio>
#include "skinnyqr/perf_model.hpp"
using namespace skinnyqr;
int main() {
  auto h = *find_hardware("H100");
  assert(intensity(Kernel::tsmRttsmR, 16) == 6.0);
  assert(std::fabs(machine_balance(h) - 15.8) < 0.02);
  assert(std::fabs(predict_time(h, Kernel::hhqr_readwrite, 8192000, 8) * 1e3 - 0.48) < 0.01);
  assert(composite_time(h, ModelMethod::svqb2, 10000000, 8) / composite_time(h, ModelMethod::tsqr, 10000000, 8) == 2.0);
  assert(find_hardware("B200") && !find_hardware("nope"));
  std::printf("%s", format_hardware_spec(*find_hardware("B200")).c_str());
  return 0;
}
