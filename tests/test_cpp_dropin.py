"""Compiles tests/cpp/test_dropin.cpp against the drop-in C++ headers
(paper_2603_20889_b200/include/skinnyqr/*.hpp) + the C ABI.  The compile/link step runs everywhere;
executing it needs the GPU."""
import json
import subprocess
from pathlib import Path

import numpy as np
import pytest

from conftest import EPS

ROOT = Path(__file__).resolve().parents[1]
PKG = ROOT / "paper_2603_20889_b200"


@pytest.fixture(scope="module")
def dropin_binary(tmp_path_factory, sq):
    sq.load_library()
    exe = tmp_path_factory.mktemp("cpp") / "test_dropin"
    cmd = ["g++", "-std=c++17", "-O1", "-I", str(PKG / "include"), "-I", str(ROOT / "include"),
           str(ROOT / "tests" / "cpp" / "test_dropin.cpp"), "-o", str(exe), "-L", str(PKG),
           "-lskinnyqr_b200", f"-Wl,-rpath,{PKG}"]
    subprocess.run(cmd, check=True)
    return exe


def test_cpp_interface_compiles_and_links(dropin_binary):
    assert dropin_binary.exists()


@pytest.mark.gpu
def test_cpp_interface_matches_oracle(dropin_binary, oracle):
    out = json.loads(subprocess.run([str(dropin_binary)], check=True, capture_output=True, text=True).stdout)
    m, n = 3001, 7
    x = oracle.uniform_pm1(m, n, 11)
    bound = 64 * n * EPS * np.linalg.norm(x)
    r_ref = oracle.port.reference_hhqr(x)
    for key in ("tsqr_qless", "tsqr_qless_k5_b32", "cholqr2"):
        r = np.array(out[key]).reshape(n, n, order="F")
        assert np.linalg.norm(r - r_ref) <= bound, key
    c = np.array(out["tsmttsm"]).reshape(n, n, order="F")
    assert np.linalg.norm(c - x.T @ x) <= 5 * n * EPS * np.linalg.norm(x) ** 2
    sg = np.linalg.svd(x, compute_uv=False)
    assert np.allclose(out["svqb2_sigma"], sg, rtol=1e-12) and out["svqb2_rank"] == n
    e = np.arange(m, dtype=np.uint64)
    rhs = x @ np.arange(1.0, n + 1.0)
    with np.errstate(over="ignore"):
        z = np.uint64(12) + (e + np.uint64(1)) * np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    rhs = rhs + 0.25 * ((z >> np.uint64(11)).astype(np.float64) * 2.0 ** -53)
    xs_ref, res_ref = oracle.port.solve_lstsq(x, rhs, "tsqr")
    assert np.allclose(out["lstsq_x"], xs_ref, rtol=1e-10)
    assert abs(out["lstsq_residual"] - res_ref) <= 1e-10 * res_ref
    assert out["caught"] == "breakdown@1;argument;dimension;zero;"


@pytest.fixture(scope="module")
def device_binary(tmp_path_factory, sq):
    sq.load_library()
    exe = tmp_path_factory.mktemp("cpp") / "test_device"
    cmd = ["g++", "-std=c++17", "-O1", "-I", str(PKG / "include"), "-I", str(ROOT / "include"),
           str(ROOT / "tests" / "cpp" / "test_device.cpp"), "-o", str(exe), "-L", str(PKG),
           "-lskinnyqr_b200", f"-Wl,-rpath,{PKG}"]
    subprocess.run(cmd, check=True)
    return exe


def test_cpp_device_interface_compiles_and_links(device_binary):
    assert device_binary.exists()


@pytest.mark.gpu
def test_cpp_device_interface_matches_oracle(device_binary, oracle):
    """DeviceMatrix overloads (X resident in HBM) and the row-sharded forms through a caller-supplied
    all-gather (this process = rank 0 of 2, the callback serves rank 1's precomputed block)."""
    out = json.loads(subprocess.run([str(device_binary)], check=True, capture_output=True, text=True).stdout)
    m, n = 30011, 9
    x = oracle.uniform_pm1(m, n, 21)
    best = oracle.best
    bound = 64 * n * EPS * np.linalg.norm(x)
    r_ref = best.tsqr_qless(x)
    for key in ("tsqr_qless", "tsqr_qless_k7_b64", "cholqr2", "tsqr_qless_sharded"):
        r = np.array(out[key]).reshape(n, n, order="F")
        assert np.linalg.norm(r - r_ref) <= bound, key
        assert np.all(np.tril(r, -1) == 0.0) and np.all(np.diag(r) >= 0.0)
    c = np.array(out["tsmttsm"]).reshape(n, n, order="F")
    assert np.linalg.norm(c - best.tsmttsm(x)) <= 5 * n * EPS * np.linalg.norm(x) ** 2
    assert np.allclose(out["svqb2_sigma"], np.linalg.svd(x, compute_uv=False), rtol=1e-12) and out["svqb2_rank"] == n
    assert np.array_equal(np.array(out["roundtrip"]), x.ravel(order="F")[:16])
    e = np.arange(m, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(22) + (e + np.uint64(1)) * np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    rhs = x @ np.arange(1.0, n + 1.0) + 0.125 * ((z >> np.uint64(11)).astype(np.float64) * 2.0 ** -53)
    xs_ref, res_ref = best.solve_lstsq(x, rhs, "tsqr")
    for kx, kr in (("lstsq_x", "lstsq_residual"), ("lstsq_sharded_x", "lstsq_sharded_residual")):
        assert np.allclose(out[kx], xs_ref, rtol=1e-10), kx
        assert abs(out[kr] - res_ref) <= 1e-10 * res_ref, kr
    assert out["exchange_calls"] == 2
