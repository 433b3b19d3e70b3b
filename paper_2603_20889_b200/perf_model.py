"""Roofline performance model of the reference (declared in include/skinnyqr/perf_model.hpp:15-74,
specified in SPEC.md "perf-model"; the reference ships the declarations only).

Pure arithmetic, no device needed.  Adds a B200 entry (measured on this pool) to the paper's Table 1
database so that bench.py can print model_time_s / model_ratio beside every measured number.
"""
from __future__ import annotations

from dataclasses import dataclass, fields

KERNELS = ("tsmttsm", "tsmRttsmR", "tsmmttsmm", "tsqr", "hhqr_readwrite")
METHODS = ("cholqr2", "svqb2", "svqb2_naive", "tsqr")


@dataclass
class HardwareSpec:
    """perf_model.hpp:15-27.  SI units (bytes/s, flops/s); mem_bandwidth is the measured value the
    predictions use, the theoretical number and the tensor rate are stored but unused."""
    name: str = ""
    mem_bandwidth: float = 0.0
    mem_bandwidth_theoretical: float = 0.0
    peak_fp64: float = 0.0
    peak_fp64_tensor: float = 0.0
    sm_count: float = 0.0
    shared_mem_per_unit: float = 0.0
    hbm_capacity: float = 0.0

    def validate(self):
        for f in fields(self):
            if f.name != "name" and not getattr(self, f.name) > 0:
                raise ValueError(f"HardwareSpec.{f.name} must be positive")


def kernel_bytes(kernel: str, m: int, n: int) -> float:
    """8*m*n for the single-read kernels, 16*m*n for hhqr_readwrite (perf_model.hpp:34-36)."""
    _check(kernel)
    return (16.0 if kernel == "hhqr_readwrite" else 8.0) * m * n


def kernel_flops(kernel: str, m: int, n: int) -> float:
    """2/3/4 * m*n^2 for the Gram kernels, 2*m*n^2 for tsqr and hhqr_readwrite (perf_model.hpp:38-40)."""
    _check(kernel)
    return {"tsmttsm": 2.0, "tsmRttsmR": 3.0, "tsmmttsmm": 4.0, "tsqr": 2.0, "hhqr_readwrite": 2.0}[kernel] * m * n * n


def intensity(kernel: str, n: int) -> float:
    """n/4, 3n/8, n/2, n/4, n/8 flops per byte, exact in FP64 (perf_model.hpp:42-44)."""
    _check(kernel)
    num, den = {"tsmttsm": (1, 4), "tsmRttsmR": (3, 8), "tsmmttsmm": (1, 2), "tsqr": (1, 4),
                "hhqr_readwrite": (1, 8)}[kernel]
    return num * n / den


def machine_balance(hw: HardwareSpec) -> float:
    return hw.peak_fp64 / hw.mem_bandwidth


def roofline_rate(hw: HardwareSpec, i: float) -> float:
    return min(hw.peak_fp64, i * hw.mem_bandwidth)


def predict_time(hw: HardwareSpec, kernel: str, m: int, n: int) -> float:
    """Memory-bound cases (I < M) are bytes/bandwidth exactly, compute-bound ones flops/peak
    (perf_model.hpp:52-54)."""
    if intensity(kernel, n) < machine_balance(hw):
        return kernel_bytes(kernel, m, n) / hw.mem_bandwidth
    return kernel_flops(kernel, m, n) / hw.peak_fp64


def composite_time(hw: HardwareSpec, method: str, m: int, n: int) -> float:
    """perf_model.hpp:56-64: cholqr2 = tsmttsm + tsmRttsmR, svqb2 = tsmttsm + tsmmttsmm,
    svqb2_naive = tsmttsm + explicit X*B pass (16mn bytes, 2mn^2 flops) + tsmttsm, tsqr = one kernel."""
    if method == "cholqr2":
        return predict_time(hw, "tsmttsm", m, n) + predict_time(hw, "tsmRttsmR", m, n)
    if method == "svqb2":
        return predict_time(hw, "tsmttsm", m, n) + predict_time(hw, "tsmmttsmm", m, n)
    if method == "svqb2_naive":
        return 2.0 * predict_time(hw, "tsmttsm", m, n) + predict_time(hw, "hhqr_readwrite", m, n)
    if method == "tsqr":
        return predict_time(hw, "tsqr", m, n)
    raise ValueError(f"unknown method {method!r}")


def _check(kernel):
    if kernel not in KERNELS:
        raise ValueError(f"unknown kernel {kernel!r}")


def hardware_database():
    """The paper's Table 1 (H100 predicts with the measured 2.15e12 B/s, the others
    ship theoretical values in both bandwidth fields) plus the B200 this repository was measured on
    (MEASURED_PEAKS.json copy bandwidth; FP64 rates from tools/probe_fp64.cu / tools/probe.cu)."""
    kb, gb = 1024.0, 1e9
    return [
        HardwareSpec("H100", 2.15e12, 3.4e12, 34e12, 67e12, 132, 228 * kb, 80 * gb),
        HardwareSpec("B100", 8.0e12, 8.0e12, 30e12, 40e12, 160, 228 * kb, 192 * gb),
        HardwareSpec("MI300X", 5.3e12, 5.3e12, 82e12, 163e12, 304, 64 * kb, 192 * gb),
        HardwareSpec("MI350X", 8.0e12, 8.0e12, 72e12, 144e12, 256, 64 * kb, 288 * gb),
        HardwareSpec("B200", 6.535e12, 8.0e12, 36.9e12, 37.1e12, 148, 227 * kb, 180 * gb),
    ]


def find_hardware(name: str):
    for hw in hardware_database():
        if hw.name == name:
            return hw
    return None


def load_hardware_spec(path: str) -> HardwareSpec:
    """Plain-text spec file: "key = value" lines, keys exactly the HardwareSpec field names, '#'
    comments and blank lines allowed (perf_model.hpp:71-73)."""
    hw = HardwareSpec()
    names = {f.name for f in fields(HardwareSpec)}
    for raw in open(path, encoding="utf-8"):
        line = raw.split("#", 1)[0].strip()
        if not line:
            continue
        key, _, val = line.partition("=")
        key, val = key.strip(), val.strip()
        if key not in names:
            raise ValueError(f"unknown HardwareSpec key {key!r}")
        setattr(hw, key, val if key == "name" else float(val))
    hw.validate()
    return hw


def format_hardware_spec(hw: HardwareSpec) -> str:
    return "".join(f"{f.name} = {getattr(hw, f.name)!r}\n".replace("'", "") for f in fields(hw))
