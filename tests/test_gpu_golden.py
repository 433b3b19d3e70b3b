"""GPU parity against the committed golden vectors (tests/golden/reference_vectors.npz: outputs of the
UNMODIFIED reference, tests/golden/make_golden.py) and on BASELINE config C1 (1 000 000 x 8), all
through the C ABI.  The golden inputs are regenerated bit-exactly from the reference's mix64 stream
(oracle.uniform_pm1), so nothing here needs /root/reference."""
from pathlib import Path

import numpy as np
import pytest

from conftest import EPS, r_bound

pytestmark = pytest.mark.gpu
GOLD = np.load(Path(__file__).parent / "golden" / "reference_vectors.npz")
CASES = [(257, 1, 3, 16), (300, 3, 2, 8), (1000, 8, 4, 32), (777, 5, 7, 10), (640, 16, 3, 40),
         (500, 32, 2, 64), (400, 64, 1, 128)]


@pytest.mark.parametrize("m,n,k,b", CASES)
def test_golden_inputs_through_the_abi(ctx, oracle, sq, m, n, k, b):
    x = oracle.uniform_pm1(m, n, 1000 + n)
    tag = f"{m}x{n}_k{k}_b{b}"
    plan = sq.PanelPlan(k, b)
    bound = r_bound(x)
    xn2 = np.linalg.norm(x) ** 2
    # TSQR family, same explicit plan as the reference run
    assert np.linalg.norm(ctx.tsqr_qless(x, plan) - GOLD[f"tsqr_qless_{tag}"]) <= bound
    assert np.linalg.norm(ctx.tsqr_qless(x) - GOLD[f"reference_hhqr_{tag}"]) <= bound
    y = ctx.tsqr_stage1(x, plan)
    yg = GOLD[f"tsqr_stage1_{tag}"]
    assert y.shape == yg.shape
    for blk in range(k):  # per-block triangles: same row partition, signs are free
        a, g = y[blk * n:(blk + 1) * n], yg[blk * n:(blk + 1) * n]
        assert np.linalg.norm(np.abs(a) - np.abs(g)) <= bound, blk
    assert np.linalg.norm(np.abs(ctx.block_qless_qr(x, b)) - np.abs(GOLD[f"block_qless_qr_{tag}"])) <= bound
    # Gram kernels
    c = ctx.tsmttsm(x, plan)
    assert np.linalg.norm(c - GOLD[f"tsmttsm_{tag}"]) <= 5 * n * EPS * xn2
    r1 = ctx.cholesky(GOLD[f"tsmttsm_{tag}"])
    assert np.linalg.norm(r1 - GOLD[f"cholesky_{tag}"]) <= 64 * n * EPS * np.sqrt(xn2)
    g2 = ctx.tsmRttsmR(x, GOLD[f"cholesky_{tag}"], plan)
    assert np.linalg.norm(g2 - GOLD[f"tsmRttsmR_{tag}"]) <= 1e-12 * n
    bm = oracle.uniform_pm1(n, n, 77)
    g3 = ctx.tsmmttsmm(x, bm, plan)
    assert np.linalg.norm(g3 - GOLD[f"tsmmttsmm_{tag}"]) <= 5 * n * EPS * np.linalg.norm(x @ bm) ** 2 + 1e-13
    assert np.linalg.norm(ctx.cholqr2(x, plan) - GOLD[f"cholqr2_{tag}"]) <= bound
    if n <= 32:
        vals, _ = ctx.eigh_small(GOLD[f"tsmttsm_{tag}"])
        assert np.allclose(vals, GOLD[f"eigh_values_{tag}"], rtol=0, atol=10 * n * EPS * xn2)
        tr, z, sg, rank = ctx.svqb2(x, plan)
        assert rank == int(GOLD[f"svqb2_rank_{tag}"][0])
        assert np.allclose(sg, GOLD[f"svqb2_sigma_{tag}"], rtol=1e-10, atol=1e-13)
        # bases are not unique; Z^T Z = C is
        zg = GOLD[f"svqb2_z_{tag}"]
        assert np.linalg.norm(z.T @ z - zg.T @ zg) <= 50 * n * EPS * xn2


def test_golden_least_squares(ctx, oracle):
    a = oracle.uniform_pm1(900, 6, 21)
    rhs = a @ np.arange(1.0, 7.0) + 0.125 * oracle.uniform_pm1(900, 1, 22)[:, 0]
    for meth in ("tsqr", "cholqr2", "svqb2"):
        xs, res = ctx.solve_lstsq(a, rhs, meth)
        assert np.allclose(xs, GOLD[f"lstsq_{meth}_x"], rtol=1e-10, atol=1e-12), meth
        assert abs(res - float(GOLD[f"lstsq_{meth}_res"][0])) <= 1e-10 * res, meth


def test_golden_conditioning_behaviour(ctx, oracle, sq):
    """Which condition numbers break CholQR2, and SVQB2's rank, as the reference recorded them
    (generate(4000, 32, kappa, 42) is restated bit-compatibly in the oracle port)."""
    for kp, st, rk in zip(GOLD["cond_kappas"], GOLD["cond_cholqr2_status"], GOLD["cond_svqb2_rank"]):
        x = oracle.port.generate(4000, 32, float(kp), 42)
        if st == 0:
            ctx.cholqr2(x, sq.PanelPlan(4, 128))
        else:
            with pytest.raises(sq.BreakdownError):
                ctx.cholqr2(x, sq.PanelPlan(4, 128))
        rank = ctx.svqb2(x, sq.PanelPlan(4, 128))[3]
        assert abs(rank - int(rk)) <= 2  # truncation threshold: +-1..2 near the edge
        r = ctx.tsqr_qless(x)            # the stable method never fails
        assert np.linalg.norm(r - oracle.best.reference_hhqr(x)) <= r_bound(x)


def test_config_c1_million_by_eight(ctx, oracle):
    """BASELINE configs[0]: Q-less TSQR and CholQR2 of a 1 000 000 x 8 Gaussian (seed 1234), generated
    on the device, copied back once and factored by the reference itself (oracle.ref) on the same bits."""
    m, n = 1_000_000, 8
    x = ctx.fill_gaussian(m, n, seed=1234)
    r_t = ctx.tsqr_qless(x)
    r_c = ctx.cholqr2(x)
    ctx.synchronize()
    xh = np.asfortranarray(x.cpu().numpy())
    best = oracle.best
    bound = r_bound(xh)
    r_ref = best.tsqr_qless(xh)
    assert np.linalg.norm(r_t.cpu().numpy() - r_ref) <= bound
    assert np.linalg.norm(r_t.cpu().numpy() - best.reference_hhqr(xh)) <= bound
    assert np.linalg.norm(r_c.cpu().numpy() - best.cholqr2(xh)) <= bound
    assert np.linalg.norm(r_c.cpu().numpy() - r_ref) <= bound
    # host-pointer route (the drop-in path) on the same matrix
    assert np.linalg.norm(ctx.tsqr_qless(xh) - r_ref) <= bound
    assert np.linalg.norm(ctx.cholqr2(xh) - r_ref) <= bound
