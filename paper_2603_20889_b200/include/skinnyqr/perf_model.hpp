// skinnyqr-b200: the Roofline model of the reference (include/skinnyqr/perf_model.hpp:15-74).  The
// reference ships these declarations without an implementation; here they are header-only so that a
// user of the drop-in headers links nothing extra.  Same names, argument meaning and error behaviour
// (ArgumentError for invalid specs / unknown names); the database adds the B200 this repository was
// measured on to the paper's Table 1.
#pragma once

#include <cstdint>
#include <fstream>
#include <optional>
#include <sstream>
#include <string>
#include <vector>

#include "skinnyqr/types.hpp"

namespace skinnyqr {

struct HardwareSpec {
  std::string name;
  double mem_bandwidth = 0;              // measured: the value predictions use
  double mem_bandwidth_theoretical = 0;
  double peak_fp64 = 0;                  // vector FMA
  double peak_fp64_tensor = 0;
  double sm_count = 0;
  double shared_mem_per_unit = 0;        // bytes
  double hbm_capacity = 0;               // bytes

  void validate() const {
    const double v[] = {mem_bandwidth, mem_bandwidth_theoretical, peak_fp64, peak_fp64_tensor,
                        sm_count, shared_mem_per_unit, hbm_capacity};
    for (double x : v)
      if (!(x > 0)) throw ArgumentError("HardwareSpec: every field must be positive");
  }
};

enum class Kernel { tsmttsm, tsmRttsmR, tsmmttsmm, tsqr, hhqr_readwrite };
enum class ModelMethod { cholqr2, svqb2, svqb2_naive, tsqr };

inline double kernel_bytes(Kernel k, std::uint64_t m, std::uint64_t n) {
  return (k == Kernel::hhqr_readwrite ? 16.0 : 8.0) * static_cast<double>(m) * static_cast<double>(n);
}

inline double kernel_flops(Kernel k, std::uint64_t m, std::uint64_t n) {
  const double c = k == Kernel::tsmRttsmR ? 3.0 : (k == Kernel::tsmmttsmm ? 4.0 : 2.0);
  return c * static_cast<double>(m) * static_cast<double>(n) * static_cast<double>(n);
}

inline double intensity(Kernel k, std::uint64_t n) {
  const double x = static_cast<double>(n);
  switch (k) {
    case Kernel::tsmttsm: return x / 4.0;
    case Kernel::tsmRttsmR: return 3.0 * x / 8.0;
    case Kernel::tsmmttsmm: return x / 2.0;
    case Kernel::tsqr: return x / 4.0;
    default: return x / 8.0;
  }
}

inline double machine_balance(const HardwareSpec& hw) { return hw.peak_fp64 / hw.mem_bandwidth; }

inline double roofline_rate(const HardwareSpec& hw, double i) {
  const double mem = i * hw.mem_bandwidth;
  return mem < hw.peak_fp64 ? mem : hw.peak_fp64;
}

inline double predict_time(const HardwareSpec& hw, Kernel k, std::uint64_t m, std::uint64_t n) {
  if (intensity(k, n) < machine_balance(hw)) return kernel_bytes(k, m, n) / hw.mem_bandwidth;
  return kernel_flops(k, m, n) / hw.peak_fp64;
}

inline double composite_time(const HardwareSpec& hw, ModelMethod method, std::uint64_t m, std::uint64_t n) {
  switch (method) {
    case ModelMethod::cholqr2:
      return predict_time(hw, Kernel::tsmttsm, m, n) + predict_time(hw, Kernel::tsmRttsmR, m, n);
    case ModelMethod::svqb2:
      return predict_time(hw, Kernel::tsmttsm, m, n) + predict_time(hw, Kernel::tsmmttsmm, m, n);
    case ModelMethod::svqb2_naive:
      return 2.0 * predict_time(hw, Kernel::tsmttsm, m, n) + predict_time(hw, Kernel::hhqr_readwrite, m, n);
    case ModelMethod::tsqr:
      return predict_time(hw, Kernel::tsqr, m, n);
  }
  throw ArgumentError("composite_time: unknown method");
}

inline const std::vector<HardwareSpec>& hardware_database() {
  static const std::vector<HardwareSpec> db = {
      {"H100", 2.15e12, 3.4e12, 34e12, 67e12, 132, 228.0 * 1024, 80e9},
      {"B100", 8.0e12, 8.0e12, 30e12, 40e12, 160, 228.0 * 1024, 192e9},
      {"MI300X", 5.3e12, 5.3e12, 82e12, 163e12, 304, 64.0 * 1024, 192e9},
      {"MI350X", 8.0e12, 8.0e12, 72e12, 144e12, 256, 64.0 * 1024, 288e9},
      {"B200", 6.535e12, 8.0e12, 36.9e12, 37.1e12, 148, 227.0 * 1024, 180e9},  // measured on this pool
  };
  return db;
}

inline std::optional<HardwareSpec> find_hardware(const std::string& name) {
  for (const HardwareSpec& hw : hardware_database())
    if (hw.name == name) return hw;
  return std::nullopt;
}

inline HardwareSpec load_hardware_spec(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw ArgumentError("load_hardware_spec: cannot open " + path);
  HardwareSpec hw;
  std::string line;
  auto trim = [](std::string s) {
    const auto a = s.find_first_not_of(" \t\r"), b = s.find_last_not_of(" \t\r");
    return a == std::string::npos ? std::string() : s.substr(a, b - a + 1);
  };
  while (std::getline(in, line)) {
    line = trim(line.substr(0, line.find('#')));
    if (line.empty()) continue;
    const auto eq = line.find('=');
    if (eq == std::string::npos) throw ArgumentError("load_hardware_spec: expected key = value");
    const std::string key = trim(line.substr(0, eq)), val = trim(line.substr(eq + 1));
    double* slot = key == "mem_bandwidth" ? &hw.mem_bandwidth
                 : key == "mem_bandwidth_theoretical" ? &hw.mem_bandwidth_theoretical
                 : key == "peak_fp64" ? &hw.peak_fp64
                 : key == "peak_fp64_tensor" ? &hw.peak_fp64_tensor
                 : key == "sm_count" ? &hw.sm_count
                 : key == "shared_mem_per_unit" ? &hw.shared_mem_per_unit
                 : key == "hbm_capacity" ? &hw.hbm_capacity : nullptr;
    if (key == "name") hw.name = val;
    else if (slot) *slot = std::stod(val);
    else throw ArgumentError("load_hardware_spec: unknown key " + key);
  }
  hw.validate();
  return hw;
}

inline std::string format_hardware_spec(const HardwareSpec& hw) {
  std::ostringstream os;
  os.precision(17);
  os << "name = " << hw.name << "\nmem_bandwidth = " << hw.mem_bandwidth
     << "\nmem_bandwidth_theoretical = " << hw.mem_bandwidth_theoretical << "\npeak_fp64 = " << hw.peak_fp64
     << "\npeak_fp64_tensor = " << hw.peak_fp64_tensor << "\nsm_count = " << hw.sm_count
     << "\nshared_mem_per_unit = " << hw.shared_mem_per_unit << "\nhbm_capacity = " << hw.hbm_capacity << "\n";
  return os.str();
}

}  // namespace skinnyqr
