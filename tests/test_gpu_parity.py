"""GPU parity tests: the CUDA path (through the C ABI, via the Python mirror of the reference
interface) against the CPU oracle on identical seeded inputs.  Tolerances are the ones DESIGN.md
states: R within 64*n*eps*|X|_F after sign normalisation, Gram within 5*n*eps*|X|_F^2."""
import numpy as np
import pytest

from conftest import EPS, gaussian, normalize, r_bound

pytestmark = pytest.mark.gpu

SHAPES = [(1000, 1), (5000, 3), (20000, 8), (4097, 5), (50000, 12), (30000, 16), (20011, 24),
          (20000, 32), (9000, 40), (8000, 56), (10000, 64), (64, 64), (130, 7)]


@pytest.mark.parametrize("m,n", SHAPES)
def test_tsqr_qless_host_matches_oracle(ctx, oracle, m, n):
    x = gaussian(m, n, seed=m + n)
    r = ctx.tsqr_qless(x)
    best = oracle.ref or oracle.port
    r_ref = best.tsqr_qless(x)
    r_hh = oracle.best.reference_hhqr(x)
    assert np.all(np.tril(r, -1) == 0.0)
    assert np.all(np.diag(r) >= 0.0)
    assert np.linalg.norm(r - r_ref) <= r_bound(x)
    assert np.linalg.norm(r - r_hh) <= r_bound(x)


@pytest.mark.parametrize("k,b", [(1, 64), (2, 24), (13, 48), (64, 16), (7, 33), (300, 8)])
def test_tsqr_plan_invariance(ctx, oracle, sq, k, b):
    x = gaussian(5000, 12, seed=3)
    r = ctx.tsqr_qless(x, sq.PanelPlan(k, b))
    r_hh = oracle.best.reference_hhqr(x)
    assert np.linalg.norm(r - r_hh) <= r_bound(x)


def test_tsqr_stage1_blocks(ctx, oracle, sq):
    x = gaussian(6000, 9, seed=11)
    plan = sq.PanelPlan(5, 64)
    y = ctx.tsqr_stage1(x, plan)
    y_ref = oracle.best.tsqr_stage1(x, 5, 64)
    assert y.shape == y_ref.shape == (45, 9)
    for blk in range(5):
        a = normalize(y[blk * 9:(blk + 1) * 9])
        b_ = normalize(y_ref[blk * 9:(blk + 1) * 9])
        lo, hi = plan.block_begin(6000, blk), plan.block_end(6000, blk)
        assert np.linalg.norm(a - b_) <= r_bound(x[lo:hi])


def test_block_qless_qr(ctx, oracle):
    x = gaussian(3000, 10, seed=5)
    r = normalize(ctx.block_qless_qr(x, 128))
    r_ref = normalize(oracle.best.block_qless_qr(x, 128))
    assert np.linalg.norm(r - r_ref) <= r_bound(x)


def test_zero_column_gives_exact_zero_row(ctx):
    x = gaussian(600, 3, seed=1)
    x[:, 1] = 0.0
    r = ctx.tsqr_qless(x)
    assert np.all(r[1, :] == 0.0)
    assert r[0, 1] == 0.0


def test_spec_examples(ctx):
    r = ctx.tsqr_qless(np.array([[1.0, 1.0], [0.0, 1.0], [0.0, 0.0]]))
    assert np.allclose(r, [[1.0, 1.0], [0.0, 1.0]], atol=1e-15)
    r = ctx.tsqr_qless(np.array([[0.0, 1.0], [1.0, 0.0]]))
    assert np.allclose(r, np.eye(2), atol=1e-15)
    c = ctx.tsmttsm(np.ones((4, 2)))
    assert np.array_equal(c, [[4.0, 4.0], [4.0, 4.0]])
    r = ctx.cholesky(np.array([[4.0, 2.0], [2.0, 5.0]]))
    assert np.allclose(r, [[2.0, 1.0], [0.0, 2.0]], atol=1e-15)
    r = ctx.cholqr2(np.array([[2.0, 0.0], [0.0, 3.0], [0.0, 0.0]]))
    assert np.allclose(r, np.diag([2.0, 3.0]), atol=1e-14)
    vals, vecs = ctx.eigh_small(np.array([[2.0, 1.0], [1.0, 2.0]]))
    assert np.allclose(vals, [3.0, 1.0], atol=1e-15)
    assert np.allclose(np.abs(vecs), np.full((2, 2), 1 / np.sqrt(2)), atol=1e-15)
    xs, res = ctx.solve_lstsq(np.ones((3, 1)), np.array([1.0, 2.0, 3.0]))
    assert np.allclose(xs, [2.0], atol=1e-15) and abs(res - np.sqrt(2.0)) < 1e-14


def test_errors(ctx, sq):
    with pytest.raises(sq.ArgumentError):
        ctx.tsqr_qless(gaussian(200, 65))
    with pytest.raises(sq.DimensionError):
        ctx.tsqr_qless(gaussian(1, 3))
    x = gaussian(5000, 6)
    x[4321, 2] = np.nan
    with pytest.raises(sq.ArgumentError):
        ctx.tsqr_qless(x)
    x[4321, 2] = np.inf
    with pytest.raises(sq.ArgumentError):
        ctx.cholqr2(x)
    with pytest.raises(sq.ArgumentError):
        ctx.tsmttsm(x)
    with pytest.raises(sq.BreakdownError) as ei:
        ctx.cholesky(np.array([[1.0, 1.0], [1.0, 1.0]]))
    assert ei.value.pivot_index == 1
    with pytest.raises(sq.SingularFactorError) as ei:
        ctx.tsmRttsmR(gaussian(100, 3), np.array([[1.0, 2.0, 3.0], [0.0, 0.0, 1.0], [0.0, 0.0, 2.0]]))
    assert ei.value.diagonal_index == 1
    with pytest.raises(sq.ZeroMatrixError):
        ctx.svqb2(np.zeros((50, 4)))
    # the context stays usable after an error
    r = ctx.tsqr_qless(gaussian(300, 4, seed=2))
    assert np.all(np.isfinite(r))


@pytest.mark.parametrize("m,n", [(3000, 1), (7001, 4), (20000, 8), (12000, 16), (9000, 24),
                                 (10000, 32), (6000, 48), (5000, 64)])
def test_gram_kernels(ctx, oracle, m, n):
    x = gaussian(m, n, seed=7 * n)
    xn2 = np.linalg.norm(x) ** 2
    c = ctx.tsmttsm(x)
    c_ref = oracle.best.tsmttsm(x)
    assert np.array_equal(c, c.T)
    assert np.linalg.norm(c - c_ref) <= 5 * n * EPS * xn2
    r1 = np.linalg.cholesky(c_ref).T.copy(order="F")
    c2 = ctx.tsmRttsmR(x, r1)
    c2_ref = oracle.best.tsmRttsmR(x, r1)
    assert np.linalg.norm(c2 - c2_ref) <= 50 * n * EPS * n
    bm = gaussian(n, n, seed=99) / np.sqrt(m)
    c3 = ctx.tsmmttsmm(x, bm)
    c3_ref = oracle.best.tsmmttsmm(x, bm)
    assert np.linalg.norm(c3 - c3_ref) <= 5 * n * EPS * np.linalg.norm(x @ bm) ** 2 + 1e-300


@pytest.mark.parametrize("m,n", [(4000, 65), (5003, 100), (9000, 128), (7001, 129), (6000, 200), (10007, 256),
                                 (130, 128), (17, 256)])
def test_wide_gram(ctx, sq, oracle, m, n):
    """BASELINE config 5 (n = 128 / 256): tsmttsm has no column limit in the reference
    (gram.cpp:113-121); the wide DMMA kernel against the oracle, host and device entry points."""
    import torch
    x = gaussian(m, n, seed=3 * n + m)
    xn2 = np.linalg.norm(x) ** 2
    c_ref = oracle.best.tsmttsm(x)
    c = ctx.tsmttsm(x)
    assert np.array_equal(c, c.T)
    assert np.linalg.norm(c - c_ref) <= 5 * n * EPS * xn2
    xd = torch.from_numpy(np.ascontiguousarray(x.T)).cuda().t()  # column-major device tensor
    cd = ctx.tsmttsm(xd)
    ctx.synchronize()
    assert np.linalg.norm(cd.cpu().numpy() - c_ref) <= 5 * n * EPS * xn2
    # unaligned leading dimension / odd row offset takes the synchronous fill path
    big = torch.zeros((n, m + 3), dtype=torch.float64, device="cuda")
    big[:, 1:m + 1] = xd.t()
    cu = ctx.tsmttsm(big.t()[1:m + 1, :])
    ctx.synchronize()
    assert np.linalg.norm(cu.cpu().numpy() - c_ref) <= 5 * n * EPS * xn2
    x[m // 2, n - 1] = np.inf
    with pytest.raises(sq.ArgumentError):
        ctx.tsmttsm(x)


@pytest.mark.parametrize("m,n", [(4000, 65), (5003, 100), (9000, 128), (20011, 127), (300, 128), (128, 128),
                                 (7001, 129), (6000, 200), (10007, 256), (300, 256), (40000, 256)])
def test_wide_solve_gram_and_cholqr2(ctx, sq, oracle, m, n):
    """64 < n <= 256: the reference's tsmRttsmR / cholqr2 / cholesky have no column limit (gram.cpp:123-140,
    gram_qr.cpp:36-58, 123-131; BASELINE config 5 names n = 128 / 256); fused solve + Gram DMMA kernel
    (explicit R^-1 GEMM feeding the SYRK; beyond 128 columns per row slab through 128 x 128 factor blocks)
    against the oracle, host and device entry points, aligned and unaligned staging, error parity."""
    import torch
    x = gaussian(m, n, seed=5 * n + m)
    c_ref = oracle.best.tsmttsm(x)
    r1 = np.linalg.cholesky(c_ref).T.copy(order="F")
    c2_ref = oracle.best.tsmRttsmR(x, r1)
    c2 = ctx.tsmRttsmR(x, r1)
    assert np.array_equal(c2, c2.T)
    assert np.linalg.norm(c2 - c2_ref) <= 50 * n * EPS * n
    assert np.linalg.norm(c2 - np.eye(n)) <= 1e-10 * np.linalg.cond(r1)
    xd = torch.from_numpy(np.ascontiguousarray(x.T)).cuda().t()
    c2d = ctx.tsmRttsmR(xd, torch.from_numpy(np.ascontiguousarray(r1.T)).cuda().t())
    ctx.synchronize()
    assert np.linalg.norm(c2d.cpu().numpy() - c2_ref) <= 50 * n * EPS * n
    big = torch.zeros((n, m + 3), dtype=torch.float64, device="cuda")
    big[:, 1:m + 1] = xd.t()
    c2u = ctx.tsmRttsmR(big.t()[1:m + 1, :], torch.from_numpy(np.ascontiguousarray(r1.T)).cuda().t())
    ctx.synchronize()
    assert np.linalg.norm(c2u.cpu().numpy() - c2_ref) <= 50 * n * EPS * n
    # a general (non-Cholesky) upper factor with a graded diagonal
    rg = np.triu(gaussian(n, n, seed=n)) / np.sqrt(n) + np.diag(np.linspace(1.0, 3.0, n))
    rg = np.asfortranarray(rg)
    cg = ctx.tsmRttsmR(x, rg)
    cg_ref = oracle.best.tsmRttsmR(x, rg)
    assert np.linalg.norm(cg - cg_ref) <= 50 * n * EPS * np.linalg.norm(cg_ref) * np.linalg.cond(rg)
    # CholQR2
    xn = np.linalg.norm(x)
    r = ctx.cholqr2(x)
    r_ref = oracle.best.cholqr2(x)
    # reconstruct_q (gram_qr.cpp:193-221) through the same solve GEMM
    q = ctx.reconstruct_q(x, r)
    q_ref = oracle.best.reconstruct_q(x, r_ref)
    assert np.linalg.norm(q - q_ref) <= 1e-11 * np.sqrt(n)
    assert np.linalg.norm(q.T @ q - np.eye(n)) <= 1e-12
    qd = ctx.reconstruct_q(xd, torch.from_numpy(np.ascontiguousarray(r.T)).cuda().t())
    ctx.synchronize()
    assert np.array_equal(qd.cpu().numpy(), q)
    assert np.all(np.tril(r, -1) == 0.0) and np.all(np.diag(r) > 0.0)
    assert np.linalg.norm(r - r_ref) <= 64 * n * EPS * xn
    assert np.linalg.norm(r.T @ r - c_ref) <= 50 * n * EPS * xn ** 2
    rd = ctx.cholqr2(xd)
    ctx.synchronize()
    assert np.linalg.norm(rd.cpu().numpy() - r_ref) <= 64 * n * EPS * xn
    # error parity: singular factor (gram.cpp:126-134) and Cholesky breakdown (gram_qr.cpp:39-54)
    rs = r1.copy(order="F")
    rs[n // 2, n // 2] = 0.0
    with pytest.raises(sq.SingularFactorError) as ei:
        ctx.tsmRttsmR(x, rs)
    assert ei.value.diagonal_index == n // 2
    xb = x.copy(order="F")
    xb[:, n - 1] = xb[:, 0]
    with pytest.raises(sq.BreakdownError):
        ctx.cholqr2(xb)
    r_again = ctx.cholqr2(x)
    assert np.array_equal(r_again, r)


@pytest.mark.parametrize("m,n", [(4000, 65), (5003, 100), (9000, 128), (20011, 127), (300, 128), (7001, 129),
                                 (6000, 200), (10007, 256)])
def test_wide_multiply_gram_and_svqb2(ctx, sq, oracle, m, n):
    """64 < n <= 128: tsmmttsmm (gram.cpp:142-151) and svqb2 (gram_qr.cpp:178-191; eigh_small's own
    limit is 128 columns, gram_qr.cpp:62) through the fused multiply + Gram DMMA kernel."""
    import torch
    x = gaussian(m, n, seed=11 * n + m)
    bm = np.asfortranarray(gaussian(n, n, seed=99) / np.sqrt(m))
    c3_ref = oracle.best.tsmmttsmm(x, bm)
    tol = 5 * n * EPS * np.linalg.norm(x @ bm) ** 2
    c3 = ctx.tsmmttsmm(x, bm)
    assert np.array_equal(c3, c3.T)
    assert np.linalg.norm(c3 - c3_ref) <= tol
    xd = torch.from_numpy(np.ascontiguousarray(x.T)).cuda().t()
    bd = torch.from_numpy(np.ascontiguousarray(bm.T)).cuda().t()
    c3d = ctx.tsmmttsmm(xd, bd)
    ctx.synchronize()
    assert np.linalg.norm(c3d.cpu().numpy() - c3_ref) <= tol
    big = torch.zeros((n, m + 3), dtype=torch.float64, device="cuda")
    big[:, 1:m + 1] = xd.t()
    c3u = ctx.tsmmttsmm(big.t()[1:m + 1, :], bd)
    ctx.synchronize()
    assert np.linalg.norm(c3u.cpu().numpy() - c3_ref) <= tol
    bad = bm.copy(order="F")
    bad[n - 1, n - 2] = np.nan
    with pytest.raises(sq.ArgumentError):
        ctx.tsmmttsmm(x, bad)
    if n > 128:  # eigh_small's own limit (gram_qr.cpp:62)
        with pytest.raises(sq.ArgumentError):
            ctx.svqb2(x)
        return
    # SVQB2
    tr, z, sg, rank = ctx.svqb2(x)
    tr_ref, z_ref, sg_ref, rank_ref = oracle.best.svqb2(x)
    assert rank == rank_ref == n
    assert np.linalg.norm(sg - sg_ref) <= 50 * n * EPS * sg_ref[0]
    c = x.T @ x
    assert np.linalg.norm(tr.T @ c @ tr - np.eye(n)) <= 1e-11
    assert np.linalg.norm(z @ tr - np.eye(n)) <= 1e-11
    assert np.linalg.norm(z.T @ z - c) <= 100 * n * EPS * np.linalg.norm(c)
    trd, zd, sgd, rankd = ctx.svqb2(xd)
    ctx.synchronize()
    assert int(rankd) == n
    assert np.linalg.norm(sgd.cpu().numpy() - sg_ref) <= 50 * n * EPS * sg_ref[0]


def test_wide_gram_limit(ctx, sq):
    with pytest.raises(sq.ArgumentError):
        ctx.svqb2(gaussian(300, 129))
    with pytest.raises(sq.ArgumentError):
        ctx.cholqr2(gaussian(300, 257))
    with pytest.raises(sq.ArgumentError):
        ctx.tsmRttsmR(gaussian(300, 257), np.eye(257))
    with pytest.raises(sq.ArgumentError):
        ctx.tsmttsm(gaussian(300, 257))


@pytest.mark.parametrize("n", [1, 2, 5, 8, 17, 32, 64, 128, 129, 200, 256])
def test_cholesky_and_eigh(ctx, sq, oracle, n):
    a = gaussian(4 * n + 3, n, seed=n)
    c = np.asfortranarray(a.T @ a)
    r = ctx.cholesky(c)
    r_ref = oracle.best.cholesky(c)
    assert np.all(np.tril(r, -1) == 0.0)
    assert np.linalg.norm(r - r_ref) <= 50 * n * EPS * np.linalg.norm(r_ref) * np.linalg.cond(c) ** 0.5
    if n > 1:  # breakdown parity: same pivot index as the reference (gram_qr.cpp:39-54)
        cb = c.copy(order="F")
        k = n // 2
        cb[k, :] = cb[k - 1, :]
        cb[:, k] = cb[:, k - 1]
        with pytest.raises(sq.BreakdownError) as ei:
            ctx.cholesky(cb)
        with pytest.raises(oracle.OracleError) as eo:
            oracle.best.cholesky(cb)
        assert ei.value.pivot_index == eo.value.index == k
    if n > 128:
        return
    vals, vecs = ctx.eigh_small(c)
    vals_ref, _ = oracle.best.eigh_small(c)
    assert np.all(np.diff(vals) <= 0.0)
    assert np.linalg.norm(vals - vals_ref) <= 50 * n * EPS * np.linalg.norm(c)
    assert np.linalg.norm(vecs.T @ vecs - np.eye(n)) <= 50 * n * EPS
    assert np.linalg.norm(c @ vecs - vecs * vals) <= 50 * n * EPS * np.linalg.norm(c)


@pytest.mark.parametrize("n", [3, 4, 6, 7, 33, 65, 66, 67, 95, 125, 126, 127])
@pytest.mark.parametrize("kind", ["graded", "clustered", "rank1", "diagonal", "scaled"])
def test_eigh_special_matrices(ctx, oracle, n, kind):
    """The grouped Jacobi (index blocks of two, padding to a multiple of 4) on spectra the Gaussian Gram matrices
    do not produce; eigenvalues against the reference's cyclic Jacobi (gram_qr.cpp:60-121), vectors through the
    invariants."""
    rng = np.random.default_rng(1000 * n + len(kind))
    q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    if kind == "graded":
        lam = np.logspace(0, -12, n)
    elif kind == "clustered":
        lam = np.where(np.arange(n) % 2 == 0, 1.0, 1.0 + 1e-9) * (1.0 + np.arange(n) // 8)
    elif kind == "rank1":
        lam = np.zeros(n)
        lam[0] = 3.0
    elif kind == "diagonal":
        lam, q = np.linspace(1.0, 2.0, n)[::-1].copy(), np.eye(n)
    else:  # entries near the edge of the range (squares ~1e300, like the reference's own Frobenius norm allows)
        lam = np.logspace(0, -6, n) * 1e150
    c = (q * lam) @ q.T
    c = np.asfortranarray(0.5 * (c + c.T))
    vals, vecs = ctx.eigh_small(c)
    vals_ref, _ = oracle.best.eigh_small(c)
    scale = np.abs(lam).max()
    assert np.all(np.diff(vals) <= 0.0)
    assert np.linalg.norm(vals - vals_ref) <= 50 * n * EPS * scale
    assert np.linalg.norm(vecs.T @ vecs - np.eye(n)) <= 50 * n * EPS
    assert np.linalg.norm(c @ vecs - vecs * vals) <= 50 * n * EPS * scale
    if kind == "diagonal":  # already converged: no rotation, U = I up to the sort
        assert np.array_equal(vals, lam) and np.array_equal(np.abs(vecs), np.eye(n))


@pytest.mark.parametrize("m,n", [(4000, 3), (20000, 8), (15000, 16), (12000, 32), (9000, 64)])
def test_cholqr2_and_svqb2(ctx, oracle, m, n):
    x = gaussian(m, n, seed=m)
    r = ctx.cholqr2(x)
    r_ref = oracle.best.cholqr2(x)
    assert np.all(np.diag(r) > 0.0)
    assert np.linalg.norm(r - r_ref) <= r_bound(x)
    tr, z, sg, rank = ctx.svqb2(x)
    tr_ref, z_ref, sg_ref, rank_ref = oracle.best.svqb2(x)
    assert rank == rank_ref == n
    assert np.linalg.norm(sg - sg_ref) <= 50 * n * EPS * sg_ref[0]
    c = x.T @ x
    assert np.linalg.norm(tr.T @ c @ tr - np.eye(n)) <= 1e-12
    assert np.linalg.norm(z @ tr - np.eye(n)) <= 1e-12
    assert np.linalg.norm(z.T @ z - c) <= 100 * n * EPS * np.linalg.norm(c)


def test_svqb_pass(ctx, oracle):
    a = gaussian(300, 12, seed=8)
    c = np.asfortranarray(a.T @ a)
    b, z, sg, rank = ctx.svqb_pass(c)
    b_ref, z_ref, sg_ref, rank_ref = oracle.best.svqb_pass(c)
    assert rank == rank_ref == 12
    assert np.linalg.norm(sg - sg_ref) <= 1e-13 * sg_ref[0]
    assert np.linalg.norm(b.T @ c @ b - np.eye(12)) <= 1e-12
    assert np.linalg.norm(z @ b - np.eye(12)) <= 1e-12
    # columns agree with the reference's up to sign (well separated spectrum)
    for j in range(12):
        s = np.sign(b[:, j] @ b_ref[:, j])
        assert np.linalg.norm(b[:, j] * s - b_ref[:, j]) <= 1e-9 * np.linalg.norm(b_ref[:, j])


def test_svqb2_truncates_rank_deficient(ctx, oracle):
    x = gaussian(5000, 6, seed=4)
    x[:, 5] = x[:, 0] + x[:, 1]
    tr, z, sg, rank = ctx.svqb2(x)
    _, _, _, rank_ref = oracle.best.svqb2(x)
    assert rank == rank_ref == 5
    assert np.all(tr[:, 5] == 0.0) and np.all(z[5, :] == 0.0)


@pytest.mark.parametrize("method", ["tsqr", "cholqr2", "svqb2"])
@pytest.mark.parametrize("m,n", [(5000, 4), (7001, 8), (20000, 15), (12000, 28), (9000, 31), (8000, 63)])
def test_solve_lstsq(ctx, oracle, method, m, n):
    a = gaussian(m, n, seed=n)
    rhs = a @ np.arange(1, n + 1, dtype=np.float64) + 0.01 * gaussian(m, 1, seed=77)[:, 0]
    xs, res = ctx.solve_lstsq(a, rhs, method)
    xs_ref, res_ref = oracle.best.solve_lstsq(a, rhs, method)
    assert np.linalg.norm(xs - xs_ref) <= 1e-10 * np.linalg.norm(xs_ref)
    assert abs(res - res_ref) <= 1e-10 * res_ref


@pytest.mark.parametrize("m,n", [(9000, 64), (12000, 100), (6001, 127)])
def test_solve_lstsq_wide_gram_routes(ctx, sq, oracle, m, n):
    """[A rhs] with 65..128 columns: the CholQR2 / SVQB2 routes have no 64-column limit in the reference
    (lstsq.cpp:31-39); rhs stays a separate array (last column of the wide kernels' view)."""
    import torch
    a = gaussian(m, n, seed=n + 1)
    rhs = a @ np.arange(1, n + 1, dtype=np.float64) + 0.01 * gaussian(m, 1, seed=78)[:, 0]
    xs, res = ctx.solve_lstsq(a, rhs, "cholqr2")
    xs_ref, res_ref = oracle.best.solve_lstsq(a, rhs, "cholqr2")
    assert np.linalg.norm(xs - xs_ref) <= 1e-10 * np.linalg.norm(xs_ref)
    assert abs(res - res_ref) <= 1e-10 * res_ref
    ad = torch.from_numpy(np.ascontiguousarray(a.T)).cuda().t()
    xd, rd = ctx.solve_lstsq(ad, torch.from_numpy(rhs).cuda(), "cholqr2")
    ctx.synchronize()
    assert np.linalg.norm(xd.cpu().numpy() - xs_ref) <= 1e-10 * np.linalg.norm(xs_ref)
    assert abs(float(rd) - res_ref) <= 1e-10 * res_ref
    xv, rv = ctx.solve_lstsq(a, rhs, "svqb2")
    xv_ref, rv_ref = oracle.best.solve_lstsq(a, rhs, "svqb2")
    assert np.linalg.norm(xv - xv_ref) <= 1e-9 * np.linalg.norm(xv_ref)
    assert abs(rv - rv_ref) <= 1e-9 * rv_ref
    with pytest.raises(sq.ArgumentError):  # tsqr.cpp:188
        ctx.solve_lstsq(a, rhs, "tsqr")


def test_lstsq_rank_deficient(ctx, sq):
    a = gaussian(400, 3, seed=1)
    a[:, 2] = 0.0
    with pytest.raises(sq.RankDeficiencyError) as ei:
        ctx.solve_lstsq(a, np.ones(400))
    assert ei.value.diagonal_index == 2


def test_reconstruct_q(ctx, oracle):
    x = gaussian(7000, 10, seed=6)
    r = ctx.tsqr_qless(x)
    q = ctx.reconstruct_q(x, r)
    q_ref = oracle.best.reconstruct_q(x, r)
    assert np.linalg.norm(q - q_ref) <= 1e-13 * np.linalg.norm(q_ref)
    assert np.linalg.norm(q.T @ q - np.eye(10)) <= 1e-13


@pytest.mark.parametrize("n,method", [(8, "tsqr"), (32, "tsqr"), (16, "cholqr2"), (8, "svqb2")])
def test_device_pointer_path(ctx, oracle, n, method):
    import torch
    m = 200_000
    x = ctx.fill_gaussian(m, n, seed=1234)
    ctx.use_torch_stream()
    xh = np.asfortranarray(x.cpu().numpy())
    x_or = oracle.gaussian(m, n, 1234)
    assert np.max(np.abs(xh - x_or)) <= 1e-13  # same stream, libm vs CUDA log/cos differ by ulps
    if method == "tsqr":
        r = ctx.tsqr_qless(x)
        ctx.synchronize()
        assert np.linalg.norm(r.cpu().numpy() - oracle.best.reference_hhqr(xh)) <= r_bound(xh)
    elif method == "cholqr2":
        r = ctx.cholqr2(x)
        ctx.synchronize()
        assert np.linalg.norm(r.cpu().numpy() - oracle.best.reference_hhqr(xh)) <= r_bound(xh)
    else:
        tr, z, sg, rank = ctx.svqb2(x)
        ctx.synchronize()
        assert int(rank.item()) == n
        c = xh.T @ xh
        tr = tr.cpu().numpy()
        assert np.linalg.norm(tr.T @ c @ tr - np.eye(n)) <= 1e-12


def test_generate_matches_reference_generator(ctx, oracle):
    x = ctx.generate(5000, 12, 1e3, seed=42)
    ctx.synchronize()
    xh = x.cpu().numpy()
    x_ref = oracle.best.generate(5000, 12, 1e3, 42)
    assert np.max(np.abs(xh - x_ref)) <= 1e-14
    s = np.linalg.svd(xh, compute_uv=False)
    assert abs(s[0] / s[-1] - 1e3) <= 1e-6 * 1e3


@pytest.mark.parametrize("kappa", [1e2, 1e6, 1e10])
def test_ill_conditioned_stability(ctx, oracle, sq, kappa):
    """BASELINE config 3 at reduced m: TSQR keeps R parity at every kappa; CholQR2 breaks down
    where the reference does."""
    x = oracle.best.generate(20000, 32, kappa, 42)
    r = ctx.tsqr_qless(x)
    r_hh = oracle.best.reference_hhqr(x)
    assert np.linalg.norm(r - r_hh) <= r_bound(x)
    ref_fails = False
    try:
        r_c_ref = oracle.best.cholqr2(x)
    except oracle.OracleError as e:
        ref_fails = e.kind == "BreakdownError"
    if ref_fails:
        with pytest.raises(sq.BreakdownError):
            ctx.cholqr2(x)
    else:
        r_c = ctx.cholqr2(x)
        assert np.linalg.norm(r_c - r_c_ref) <= 64 * 32 * EPS * np.linalg.norm(x) * max(1.0, kappa * 1e-4)


def test_nccl_collective_path_single_rank(sq, oracle):
    """The sharded entry points with a real (1-rank) NCCL communicator: all-gather + combine for
    TSQR, all-reduce for the Gram methods.  More ranks need more GPUs than this box has."""
    import torch
    c = sq.Context(0)
    c.use_torch_stream()
    c.init_nccl(c.nccl_unique_id(), 0, 1)
    m, n = 300_000, 12
    x = c.fill_gaussian(m, n, seed=5)
    r = c.tsqr_qless_sharded(x)
    rc = c.cholqr2_sharded(x)
    tr, z, sg, rank = c.svqb2_sharded(x)
    rhs = torch.ones(m, dtype=torch.float64, device=x.device)
    xs, res = c.solve_lstsq_sharded(x, rhs)
    c.synchronize()
    xh = np.asfortranarray(x.cpu().numpy())
    r_ref = oracle.best.reference_hhqr(xh)
    assert np.linalg.norm(r.cpu().numpy() - r_ref) <= r_bound(xh)
    assert np.linalg.norm(rc.cpu().numpy() - r_ref) <= r_bound(xh)
    assert int(rank.item()) == n
    xs_ref, res_ref = oracle.best.solve_lstsq(xh, np.ones(m), "tsqr")
    assert np.allclose(xs.cpu().numpy(), xs_ref, rtol=1e-9, atol=1e-12)
    assert abs(float(res.item()) - res_ref) <= 1e-10 * res_ref
    c.close()


def test_large_m_self_consistency(ctx):
    """Full-size style check without the oracle: R^T R of TSQR equals the independently computed
    Gram matrix, and CholQR2's R equals TSQR's (size-independent properties)."""
    m, n = 1 << 22, 16
    x = ctx.fill_gaussian(m, n, seed=9)
    ctx.use_torch_stream()
    r = ctx.tsqr_qless(x)
    c = ctx.tsmttsm(x)
    rc = ctx.cholqr2(x)
    ctx.synchronize()
    r, c, rc = r.cpu().numpy(), c.cpu().numpy(), rc.cpu().numpy()
    xn2 = np.trace(c)
    assert np.linalg.norm(r.T @ r - c) <= 50 * n * EPS * xn2
    assert np.linalg.norm(r - rc) <= 64 * n * EPS * np.sqrt(xn2)


@pytest.mark.parametrize("n", [4, 8, 9, 12, 13, 16, 20, 31, 40, 63])
def test_device_lstsq_with_constant_rhs(ctx, oracle, n):
    """Regression: leaves with fewer rows than columns exhaust their rank in the first fold and then
    see reflector norms that underflow (1e-32, 1e-64, ... ) - the reflector scalars must not
    overflow there.  Also covers the separate-rhs device path (MatView::extra)."""
    import torch
    m = 20_000
    x = ctx.fill_gaussian(m, n, seed=5)
    ctx.use_torch_stream()
    rhs = torch.ones(m, dtype=torch.float64, device=x.device)
    for method in ("tsqr", "cholqr2"):
        xs, res = ctx.solve_lstsq(x, rhs, method)
        ctx.synchronize()
        xh = np.asfortranarray(x.cpu().numpy())
        xs_ref, res_ref = oracle.best.solve_lstsq(xh, np.ones(m), method)
        assert np.allclose(xs.cpu().numpy(), xs_ref, rtol=1e-9, atol=1e-13)
        assert abs(float(res.item()) - res_ref) <= 1e-10 * res_ref


@pytest.mark.parametrize("kind", ["thread", "fold", "mma"])
def test_every_tsqr_kernel_family(kind, sq, oracle):
    """The TSQR kernel families (thread-private leaves / lookahead fold / DMMA blocked) on the same
    inputs, forced through sqb_set_tsqr_kernel so that the measured selection table is bypassed (a
    family that cannot run a column count falls back to the table)."""
    c2 = sq.Context(0)
    c2.set_tsqr_kernel(kind)
    try:
        for m, n in [(12345, 3), (3, 3), (9002, 4), (801, 4), (9000, 5), (9001, 11), (20000, 16), (30011, 17), (7000, 24), (40000, 29), (40002, 32),
                     (6000, 33), (9000, 47), (5000, 64), (70000, 64)]:
            x = gaussian(m, n, seed=n)
            x[:, n // 2] = 1.0
            r = c2.tsqr_qless(x)
            assert np.linalg.norm(r - oracle.best.reference_hhqr(x)) <= r_bound(x), (m, n)
    finally:
        c2.close()


@pytest.mark.parametrize("n", [8, 16, 32, 64])
def test_full_size_self_consistency(ctx, n):
    """BASELINE configs[1] at its real size (m = 2^27, up to 64 GiB resident): no CPU oracle fits there,
    so parity is through size-independent properties - R^T R against the independently
    computed Gram matrix, TSQR against CholQR2, and |(X R^-1)^T (X R^-1) - I| from the fused sweep."""
    import torch
    free, _ = torch.cuda.mem_get_info()
    m = 1 << 27
    if free < 8 * m * n + (4 << 30):
        pytest.skip("not enough free HBM for the full-size matrix")
    x = ctx.fill_gaussian(m, n, seed=1234)
    r = ctx.tsqr_qless(x)
    r2 = ctx.cholqr2(x)
    c = ctx.tsmttsm(x)
    g = ctx.tsmRttsmR(x, r)
    ctx.synchronize()
    rh, r2h, ch, gh = (t.cpu().numpy() for t in (r, r2, c, g))
    xn2 = float(np.trace(ch))  # |X|_F^2
    assert np.all(np.tril(rh, -1) == 0.0) and np.all(np.diag(rh) > 0.0)
    assert np.linalg.norm(rh.T @ rh - ch) <= 50 * n * EPS * xn2
    assert np.linalg.norm(rh - r2h) <= 64 * n * EPS * np.sqrt(xn2)
    assert np.linalg.norm(gh - np.eye(n), 2) <= 1e-12
    del x
    torch.cuda.empty_cache()
