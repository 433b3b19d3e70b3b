"""Pins the CPU oracle (oracle/oracle_c.c, the C restatement) against
  (a) the SPEC worked examples the compiled reference honours,
  (b) golden vectors produced by the UNMODIFIED reference (tests/golden/make_golden.py),
  (c) the compiled reference itself when oracle/_ref is present (dev container and GPU box).
No GPU needed."""
from pathlib import Path

import numpy as np
import pytest

from conftest import EPS, normalize

GOLD = np.load(Path(__file__).parent / "golden" / "reference_vectors.npz")
CASES = [(257, 1, 3, 16), (300, 3, 2, 8), (1000, 8, 4, 32), (777, 5, 7, 10), (640, 16, 3, 40),
         (500, 32, 2, 64), (400, 64, 1, 128)]


def close(a, b, rel=1e-12):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) <= rel * max(np.linalg.norm(b), 1e-300)


def test_stream_kats(port):
    assert port.mix64(42, 0) == 0xBDD732262FEB6E95 and port.mix64(42, 1) == 0x28EFE333B266F103
    assert port.uniform01(42, 0) == 0.74156487877182331
    assert np.array_equal(np.array([port.mix64(42, i) for i in range(4)], dtype=np.uint64), GOLD["mix64_42"])
    assert np.array_equal(np.array([port.uniform01(42, i) for i in range(4)]), GOLD["uniform01_42"])


def test_generate_matches_reference(port):
    g = port.generate(5000, 12, 1e3, 42)
    assert abs(g[0, 0] - 0.052176887095362327) <= 1e-15
    assert abs(g[4999, 11] - 0.00014220804705110732) <= 1e-17
    assert np.allclose([g[0, 0], g[4999, 11], g[17, 5], g[4000, 0]],
                       GOLD["generate_5000x12_k1e3_s42_corners"], rtol=1e-12, atol=1e-16)
    assert close(port.generate(60, 5, 1e6, 7), GOLD["generate_60x5_k1e6_s7"])
    assert close(port.generate(40, 4, 50.0, 3, linear=True), GOLD["generate_40x4_lin_k50_s3"])


def test_spec_worked_examples(port, oracle):
    pen = port.factor_trapezoidal(np.array([[3.0, 0.0], [4.0, 0.0], [0.0, 1.0]]), 3)
    assert np.allclose(np.abs(pen[:2, :2]), [[5.0, 0.0], [0.0, 1.0]], atol=1e-15)
    assert close(pen, GOLD["factor_trapezoidal_spec"])
    assert np.allclose(port.reference_hhqr(np.array([[1.0, 1.0], [0.0, 1.0], [0.0, 0.0]])), [[1, 1], [0, 1]])
    assert np.allclose(port.reference_hhqr(np.array([[0.0, 1.0], [1.0, 0.0]])), np.eye(2))
    assert np.array_equal(port.tsmttsm(np.ones((4, 2)), 1, 4), [[4.0, 4.0], [4.0, 4.0]])
    assert np.allclose(port.cholesky(np.array([[4.0, 2.0], [2.0, 5.0]])), [[2.0, 1.0], [0.0, 2.0]])
    with pytest.raises(oracle.OracleError) as ei:
        port.cholesky(np.array([[1.0, 1.0], [1.0, 1.0]]))
    assert ei.value.kind == "BreakdownError" and ei.value.index == 1
    assert np.allclose(port.cholqr2(np.array([[2.0, 0.0], [0.0, 3.0], [0.0, 0.0]]), 1, 2), np.diag([2.0, 3.0]))
    vals, vecs = port.eigh_small(np.array([[2.0, 1.0], [1.0, 2.0]]))
    assert np.allclose(vals, [3.0, 1.0]) and np.allclose(np.abs(vecs), 1 / np.sqrt(2))
    xs, res = port.solve_lstsq(np.ones((3, 1)), np.array([1.0, 2.0, 3.0]))
    assert np.allclose(xs, [2.0]) and abs(res - np.sqrt(2.0)) < 1e-15
    x = np.asfortranarray(np.random.default_rng(0).standard_normal((6, 3)))
    x[:, 1] = 0.0
    r = port.tsqr_qless(x, 2, 2)
    assert np.all(r[1, :] == 0.0)
    with pytest.raises(oracle.OracleError):
        port.tsqr_qless(np.zeros((70, 65)), 1, 130)


@pytest.mark.parametrize("m,n,k,b", CASES)
def test_port_matches_golden(port, oracle, m, n, k, b):
    x = oracle.uniform_pm1(m, n, 1000 + n)
    tag = f"{m}x{n}_k{k}_b{b}"
    assert close(port.tsqr_qless(x, k, b), GOLD[f"tsqr_qless_{tag}"])
    assert close(port.tsqr_stage1(x, k, b), GOLD[f"tsqr_stage1_{tag}"])
    assert close(port.reference_hhqr(x), GOLD[f"reference_hhqr_{tag}"])
    assert close(port.block_qless_qr(x, b), GOLD[f"block_qless_qr_{tag}"])
    c = port.tsmttsm(x, k, b)
    assert close(c, GOLD[f"tsmttsm_{tag}"]) and np.array_equal(c, c.T)
    r1 = port.cholesky(GOLD[f"tsmttsm_{tag}"])
    assert close(r1, GOLD[f"cholesky_{tag}"])
    assert close(port.tsmRttsmR(x, GOLD[f"cholesky_{tag}"], k, b), GOLD[f"tsmRttsmR_{tag}"], 1e-11)
    assert close(port.tsmmttsmm(x, oracle.uniform_pm1(n, n, 77), k, b), GOLD[f"tsmmttsmm_{tag}"])
    assert close(port.cholqr2(x, k, b), GOLD[f"cholqr2_{tag}"])
    if n <= 32:
        vals, vecs = port.eigh_small(GOLD[f"tsmttsm_{tag}"])
        assert close(vals, GOLD[f"eigh_values_{tag}"])
        tr, z, sg, rank = port.svqb2(x, k, b)
        assert rank == int(GOLD[f"svqb2_rank_{tag}"][0])
        assert close(sg, GOLD[f"svqb2_sigma_{tag}"])
        bp, zp, sp, rp = port.svqb_pass(GOLD[f"tsmttsm_{tag}"])
        assert rp == int(GOLD[f"svqb_pass_rank_{tag}"][0]) and close(sp, GOLD[f"svqb_pass_sigma_{tag}"])
        # eigenvectors of a Gaussian-like Gram matrix are well separated here: compare up to sign
        gb = GOLD[f"svqb_pass_b_{tag}"]
        for j in range(n):
            s = np.sign(bp[:, j] @ gb[:, j])
            assert np.linalg.norm(bp[:, j] * s - gb[:, j]) <= 1e-8 * np.linalg.norm(gb[:, j])


def test_lstsq_and_conditioning_golden(port, oracle):
    a = oracle.uniform_pm1(900, 6, 21)
    rhs = a @ np.arange(1.0, 7.0) + 0.125 * oracle.uniform_pm1(900, 1, 22)[:, 0]
    port.threads = 4
    for meth in ("tsqr", "cholqr2", "svqb2"):
        xs, res = port.solve_lstsq(a, rhs, meth)
        assert close(xs, GOLD[f"lstsq_{meth}_x"], 1e-11) and close([res], GOLD[f"lstsq_{meth}_res"], 1e-11)
    for kp, st, rk in zip(GOLD["cond_kappas"], GOLD["cond_cholqr2_status"], GOLD["cond_svqb2_rank"]):
        x = port.generate(4000, 32, float(kp), 42)
        try:
            port.cholqr2(x, 4, 128)
            got = 0
        except oracle.OracleError as e:
            got = e.status
        assert got == int(st), (kp, got, st)
        assert abs(port.svqb2(x, 4, 128)[3] - int(rk)) <= 1
        r = port.tsqr_qless(x, 4, 128)
        assert np.linalg.norm(r - port.reference_hhqr(x)) <= 64 * 32 * EPS * np.linalg.norm(x)


def test_plans_golden(port):
    assert [port.default_tsqr_plan(10**6, n)[1] for n in (1, 8, 16, 32, 64)] == list(GOLD["default_tsqr_panel_rows"])
    assert [port.default_gram_plan(10**6, n)[1] for n in (1, 8, 16, 32, 64, 200)] == list(GOLD["default_gram_panel_rows"])
    assert [list(port.block_range(1003, 7, 16, i)) for i in range(7)] == GOLD["block_ranges_m1003_k7_b16"].tolist()


@pytest.mark.parametrize("m,n", [(3000, 4), (5000, 12), (2000, 33)])
def test_port_matches_compiled_reference(port, ref, oracle, m, n):
    x = oracle.gaussian(m, n, 7)
    k, b = 3, 4 * n
    assert close(port.tsqr_qless(x, k, b), ref.tsqr_qless(x, k, b))
    assert close(port.cholqr2(x, k, b), ref.cholqr2(x, k, b))
    assert close(port.tsmttsm(x, k, b), ref.tsmttsm(x, k, b))
    assert close(normalize(port.block_qless_qr(x, b)), normalize(ref.block_qless_qr(x, b)))
    ref.counters_reset()
    ref.tsqr_qless(x, k, b)
    assert ref.counters()["large_reads"] == m * n  # single pass over X
    ref.counters_reset()
    ref.cholqr2(x, k, b)
    assert ref.counters()["large_reads"] == 2 * m * n
