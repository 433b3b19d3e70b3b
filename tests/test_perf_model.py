"""Roofline model (reference include/skinnyqr/perf_model.hpp, SPEC.md perf-model examples)."""
import pytest

from paper_2603_20889_b200 import perf_model as pm


def test_intensity_examples():
    assert pm.intensity("tsmttsm", 8) == 2.0
    assert pm.intensity("tsmRttsmR", 16) == 6.0
    assert pm.intensity("tsmmttsmm", 32) == 16.0
    assert pm.intensity("tsqr", 8) == 2.0
    assert pm.intensity("hhqr_readwrite", 8) == 1.0
    for k in pm.KERNELS:  # independent of m: exact rational identity
        for n in (1, 3, 8, 64):
            assert pm.kernel_flops(k, 1000, n) / pm.kernel_bytes(k, 1000, n) == pm.intensity(k, n)
            assert pm.kernel_flops(k, 7, n) / pm.kernel_bytes(k, 7, n) == pm.intensity(k, n)


def test_machine_balance_and_roofline():
    h100 = pm.find_hardware("H100")
    assert pm.machine_balance(pm.HardwareSpec("x", 3.4e12, 3.4e12, 34e12, 1, 1, 1, 1)) == 10.0
    assert abs(pm.machine_balance(h100) - 15.8) < 0.02
    assert pm.roofline_rate(h100, 0.0) == 0.0
    assert pm.roofline_rate(h100, 2.0) == 4.3e12
    assert pm.roofline_rate(h100, 1e6) == 34e12


def test_predict_time_table2():
    h100 = pm.find_hardware("H100")
    for m, ms in ((8_192_000, 0.48), (81_920_000, 4.8), (819_200_000, 48.0)):
        assert abs(pm.predict_time(h100, "hhqr_readwrite", m, 8) * 1e3 - ms) <= 0.02 * ms
    assert abs(pm.predict_time(h100, "tsqr", 8_192_000, 8) * 1e3 - 0.24) < 0.005
    # memory-bound predictions are bytes / bandwidth exactly
    assert pm.predict_time(h100, "tsmttsm", 10**6, 8) == 8.0 * 10**6 * 8 / 2.15e12
    # monotone in m
    assert pm.predict_time(h100, "tsqr", 2 * 10**6, 32) >= pm.predict_time(h100, "tsqr", 10**6, 32)


def test_composite():
    h100 = pm.find_hardware("H100")
    m = 10**7
    assert pm.composite_time(h100, "svqb2", m, 8) / pm.composite_time(h100, "tsqr", m, 8) == 2.0
    assert pm.composite_time(h100, "cholqr2", m, 8) == 2 * 8.0 * m * 8 / 2.15e12
    assert pm.composite_time(h100, "svqb2_naive", m, 8) == pytest.approx(4 * 8.0 * m * 8 / 2.15e12)
    n_cb = 64  # 3n/8 = 24 > M = 15.8: the second CholQR2 sweep is compute bound on H100
    assert pm.predict_time(h100, "tsmRttsmR", m, n_cb) == 3.0 * m * n_cb * n_cb / 34e12
    with pytest.raises(ValueError):
        pm.composite_time(h100, "lu", m, 8)


def test_database_and_spec_file(tmp_path):
    names = [h.name for h in pm.hardware_database()]
    assert names[:4] == ["H100", "B100", "MI300X", "MI350X"] and "B200" in names
    for h in pm.hardware_database():
        h.validate()
    b200 = pm.find_hardware("B200")
    # the kink of Householder TSQR on B200: n/4 crosses M = 36.9/6.535 between n = 22 and 23
    assert pm.intensity("tsqr", 22) < pm.machine_balance(b200) < pm.intensity("tsqr", 23)
    p = tmp_path / "hw.txt"
    p.write_text("# comment\n" + pm.format_hardware_spec(b200) + "\n")
    assert pm.load_hardware_spec(str(p)) == b200
    p.write_text("name = x\nbogus = 1\n")
    with pytest.raises(ValueError):
        pm.load_hardware_spec(str(p))
    assert pm.find_hardware("nope") is None


def test_cpp_header_mirror(tmp_path):
    """The header-only C++ mirror (paper_2603_20889_b200/include/skinnyqr/perf_model.hpp) gives the same
    answers; it needs no CUDA library, so this runs on the CPU box."""
    import shutil
    import subprocess
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    gxx = shutil.which("g++")
    if gxx is None:
        pytest.skip("no g++")
    exe = tmp_path / "pm"
    subprocess.run([gxx, "-std=c++17", "-I", str(root / "paper_2603_20889_b200" / "include"), "-I", str(root / "include"),
                    str(root / "tests" / "cpp" / "test_perf_model.cpp"), "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout
    spec = tmp_path / "b200.txt"
    spec.write_text(out)
    assert pm.load_hardware_spec(str(spec)) == pm.find_hardware("B200")
