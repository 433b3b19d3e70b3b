"""TSKM files (reference include/skinnyqr/io.hpp, src/io.cpp) and the skinny-qr style CLI."""
import json
import struct
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

import paper_2603_20889_b200 as sq
from paper_2603_20889_b200 import io as tio

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden" / "reference_5x3.tskm"


def test_reads_file_written_by_the_reference():
    """tests/golden/reference_5x3.tskm was written by the unmodified reference (matrix_write, io.cpp:41-59;
    generator: tests/golden/make_golden_tskm.cpp, which also read back a file written by this module)."""
    x = tio.matrix_read(GOLDEN)
    i, j = np.meshgrid(np.arange(5), np.arange(3), indexing="ij")
    assert x.shape == (5, 3) and x.flags.f_contiguous
    assert np.array_equal(x, 0.5 * i - 1.25 * j + 1.0 / 3.0)
    assert tio.read_header(GOLDEN) == (5, 3)


def test_roundtrip_is_bit_exact(tmp_path):
    rng = np.random.default_rng(5)
    for shape in ((1, 1), (37, 5), (4, 9)):
        x = rng.standard_normal(shape)
        x[0, 0] = np.nextafter(1.0, 2.0)
        p = tmp_path / "x.tskm"
        tio.matrix_write(p, x)  # C-ordered input is stored in column order all the same
        assert p.stat().st_size == tio.HEADER_BYTES + 8 * x.size
        assert np.array_equal(tio.matrix_read(p), x)
        raw = p.read_bytes()
        assert raw[:4] == b"TSKM" and raw[4] == 1 and struct.unpack("<IQQ", raw[5:25]) == (8, *shape)
        assert np.array_equal(np.frombuffer(raw[25:], dtype="<f8"), x.T.ravel())


def test_error_taxonomy(tmp_path):
    """io.cpp:61-84: IoError, TruncationError, FormatError, DimensionError, SizeOverflowError."""
    p = tmp_path / "bad.tskm"
    with pytest.raises(tio.IoError):
        tio.matrix_read(tmp_path / "missing.tskm")
    p.write_bytes(b"TSK")
    with pytest.raises(tio.TruncationError):
        tio.matrix_read(p)
    hdr = lambda magic=b"TSKM", ver=1, es=8, m=2, n=2: magic + struct.pack("<BIQQ", ver, es, m, n)  # noqa: E731
    for bad in (hdr(magic=b"TSKX"), hdr(ver=2), hdr(es=4)):
        p.write_bytes(bad + bytes(32))
        with pytest.raises(tio.FormatError):
            tio.matrix_read(p)
    p.write_bytes(hdr(m=0) + bytes(32))
    with pytest.raises(sq.DimensionError):
        tio.matrix_read(p)
    p.write_bytes(hdr(m=2**62, n=8))
    with pytest.raises(tio.SizeOverflowError):
        tio.matrix_read(p)
    p.write_bytes(hdr(m=3, n=2) + bytes(40))  # 48 payload bytes announced
    with pytest.raises(tio.TruncationError):
        tio.matrix_read(p)
    for exc in (tio.IoError, tio.FormatError, tio.TruncationError, tio.SizeOverflowError):
        assert issubclass(exc, sq.Error)


def run_cli(*args):
    return subprocess.run([sys.executable, "-m", "paper_2603_20889_b200", *args], cwd=ROOT, capture_output=True, text=True)


def test_cli_model_needs_no_gpu():
    out = run_cli("model", "--hw", "H100", "--kernel", "hhqr_readwrite", "--m", "8192000", "--n", "8")
    assert out.returncode == 0, out.stderr
    assert abs(json.loads(out.stdout)["time_s"] * 1e3 - 0.48) < 0.01  # Table 2 of the paper
    out = run_cli("model", "--hw", "B200", "--kernel", "svqb2", "--m", "1000000", "--n", "8")
    t2 = json.loads(out.stdout)["time_s"]
    out = run_cli("model", "--hw", "B200", "--kernel", "tsqr", "--m", "1000000", "--n", "8")
    assert t2 / json.loads(out.stdout)["time_s"] == 2.0


def test_render_formats_agree():
    from paper_2603_20889_b200.__main__ import COLUMNS, render
    row = {c: 1.5 for c in COLUMNS}
    row.update(method="tsqr", m=10, n=2, reps=3, seed=1)
    assert render([], "csv").strip() == ",".join(COLUMNS)  # empty table -> header only
    js = json.loads(render([row], "json"))[0]
    import csv
    import io
    cs = next(csv.DictReader(io.StringIO(render([row], "csv"))))
    assert all(str(js[c]) == cs[c] for c in COLUMNS)


@pytest.mark.gpu
def test_device_stream_and_cli_end_to_end(tmp_path, oracle):
    ctx = sq.default_context(0)
    rng = np.random.default_rng(9)
    m, n = 50_003, 7
    a = np.asfortranarray(rng.standard_normal((m, n)))
    xt = np.arange(1, n + 1) / n
    b = a @ xt + 1e-3 * rng.standard_normal(m)
    tio.matrix_write(tmp_path / "a.tskm", a)
    tio.matrix_write(tmp_path / "b.tskm", b.reshape(-1, 1))
    xd = tio.matrix_read_device(tmp_path / "a.tskm", ctx, chunk_bytes=1 << 16)  # many chunks, ragged tail
    assert xd.shape == (m, n) and xd.stride() == (1, m)
    assert np.array_equal(xd.cpu().numpy(), a)
    out = run_cli("lstsq", "--matrix", str(tmp_path / "a.tskm"), "--rhs", str(tmp_path / "b.tskm"))
    assert out.returncode == 0, out.stderr
    res = json.loads(out.stdout)
    xs_ref, r_ref = oracle.port.solve_lstsq(a, b, "tsqr")
    assert np.allclose(res["x"], xs_ref, rtol=1e-9, atol=1e-12) and abs(res["residual_norm"] - r_ref) <= 1e-9 * r_ref
    out = run_cli("qr", "--matrix", str(tmp_path / "a.tskm"), "--out", str(tmp_path / "r.tskm"))
    assert out.returncode == 0, out.stderr
    r = tio.matrix_read(tmp_path / "r.tskm")
    assert np.linalg.norm(r - oracle.port.tsqr_qless(a)) <= 64 * n * np.finfo(float).eps * np.linalg.norm(a)
    out = run_cli("bench", "--mn-product", str(1 << 20), "--cols", "1,8,65,129", "--methods", "tsqr,cholqr2,svqb2",
                  "--reps", "5", "--format", "json")
    assert out.returncode == 0, out.stderr
    rows = json.loads(out.stdout)
    assert len(rows) == 12
    # TSQR stops at 64 columns (tsqr.cpp:188), SVQB2 at 128 (eigh_small, gram_qr.cpp:62), CholQR2 at 256 here
    good = [r for r in rows if r["n"] <= 8 or (r["n"] == 65 and r["method"] != "tsqr")
            or (r["n"] == 129 and r["method"] == "cholqr2")]
    assert len(good) == 9
    assert all(isinstance(r["orth_resid"], float) and r["orth_resid"] <= 1e-12 and r["model_ratio"] > 0 for r in good)
    assert all(r["large_reads"] == (1 if r["method"] == "tsqr" else 2) * r["m"] * r["n"] for r in good)
    bad = [r for r in rows if r not in good]
    assert len(bad) == 3 and all(r["orth_resid"] == "ArgumentError" for r in bad)  # per-row error, the grid continues
    assert run_cli("bench", "--reps", "0").returncode != 0


def test_cpp_io_header(tmp_path):
    """The header-only C++ mirror reads the reference-written golden file and writes a byte-identical copy."""
    import shutil
    gxx = shutil.which("g++")
    if gxx is None:
        pytest.skip("no g++")
    exe = tmp_path / "io"
    subprocess.run([gxx, "-std=c++17", "-I", str(ROOT / "paper_2603_20889_b200" / "include"), "-I", str(ROOT / "include"),
                    str(ROOT / "tests" / "cpp" / "test_io.cpp"), "-o", str(exe)], check=True)
    out = subprocess.run([str(exe), str(GOLDEN), str(tmp_path / "copy.tskm")], capture_output=True, text=True)
    assert out.returncode == 0 and "ok" in out.stdout
    assert (tmp_path / "copy.tskm").read_bytes() == GOLDEN.read_bytes()
