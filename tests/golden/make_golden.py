"""Generates tests/golden/reference_vectors.npz from the UNMODIFIED reference (oracle/_ref, built by
`make -C oracle ref` from /root/reference/proj).  Run in the build container only:

    python tests/golden/make_golden.py

Inputs are bit-reproducible (oracle.uniform_pm1: exact arithmetic on the reference's mix64 stream),
outputs are whatever the reference's own entry points return with explicit plans (k, b), so the
fixture does not depend on the host's core count.
"""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import oracle  # noqa: E402

ref = oracle.ref
assert ref is not None, "oracle/_ref/libskinnyqr_ref.so missing: run `make -C oracle ref`"
out = {}

# stream KATs
out["mix64_42"] = np.array([ref.mix64(42, i) for i in range(4)], dtype=np.uint64)
out["uniform01_42"] = np.array([ref.uniform01(42, i) for i in range(4)])
g = ref.generate(5000, 12, 1e3, 42)
out["generate_5000x12_k1e3_s42_corners"] = np.array([g[0, 0], g[4999, 11], g[17, 5], g[4000, 0]])
out["generate_60x5_k1e6_s7"] = ref.generate(60, 5, 1e6, 7)
out["generate_40x4_lin_k50_s3"] = ref.generate(40, 4, 50.0, 3, linear=True)

cases = [(257, 1, 3, 16), (300, 3, 2, 8), (1000, 8, 4, 32), (777, 5, 7, 10), (640, 16, 3, 40),
         (500, 32, 2, 64), (400, 64, 1, 128)]
for m, n, k, b in cases:
    x = oracle.uniform_pm1(m, n, 1000 + n)
    tag = f"{m}x{n}_k{k}_b{b}"
    out[f"tsqr_qless_{tag}"] = ref.tsqr_qless(x, k, b)
    out[f"tsqr_stage1_{tag}"] = ref.tsqr_stage1(x, k, b)
    out[f"reference_hhqr_{tag}"] = ref.reference_hhqr(x)
    out[f"block_qless_qr_{tag}"] = ref.block_qless_qr(x, b)
    c = ref.tsmttsm(x, k, b)
    out[f"tsmttsm_{tag}"] = c
    r1 = ref.cholesky(c)
    out[f"cholesky_{tag}"] = r1
    out[f"tsmRttsmR_{tag}"] = ref.tsmRttsmR(x, r1, k, b)
    bm = oracle.uniform_pm1(n, n, 77)
    out[f"tsmmttsmm_{tag}"] = ref.tsmmttsmm(x, bm, k, b)
    out[f"cholqr2_{tag}"] = ref.cholqr2(x, k, b)
    if n <= 32:
        vals, vecs = ref.eigh_small(c)
        out[f"eigh_values_{tag}"] = vals
        out[f"eigh_vectors_{tag}"] = vecs
        tr, z, sg, rank = ref.svqb2(x, k, b)
        out[f"svqb2_transform_{tag}"] = tr
        out[f"svqb2_z_{tag}"] = z
        out[f"svqb2_sigma_{tag}"] = sg
        out[f"svqb2_rank_{tag}"] = np.array([rank])
        bp, zp, sp, rp = ref.svqb_pass(c)
        out[f"svqb_pass_b_{tag}"] = bp
        out[f"svqb_pass_z_{tag}"] = zp
        out[f"svqb_pass_sigma_{tag}"] = sp
        out[f"svqb_pass_rank_{tag}"] = np.array([rp])

# factor_trapezoidal: SPEC example + a random pencil
out["factor_trapezoidal_spec"] = ref.factor_trapezoidal(np.array([[3.0, 0.0], [4.0, 0.0], [0.0, 1.0]]), 3)
out["factor_trapezoidal_9x4_b12"] = ref.factor_trapezoidal(oracle.uniform_pm1(9, 4, 5), 12)

# least squares (threads fixed to 4 so that the default plans inside solve_lstsq are reproducible)
ref.set_threads(4)
a = oracle.uniform_pm1(900, 6, 21)
rhs = a @ np.arange(1.0, 7.0) + 0.125 * oracle.uniform_pm1(900, 1, 22)[:, 0]
for meth in ("tsqr", "cholqr2", "svqb2"):
    xs, res = ref.solve_lstsq(a, rhs, meth)
    out[f"lstsq_{meth}_x"] = xs
    out[f"lstsq_{meth}_res"] = np.array([res])

# conditioning behaviour: which kappas break cholqr2, svqb2 ranks
kappas = [1e2, 1e6, 1e8, 1e10, 1e12]
status, ranks = [], []
for kp in kappas:
    x = ref.generate(4000, 32, kp, 42)
    try:
        ref.cholqr2(x, 4, 128)
        status.append(0)
    except oracle.OracleError as e:
        status.append(e.status)
    ranks.append(ref.svqb2(x, 4, 128)[3])
out["cond_kappas"] = np.array(kappas)
out["cond_cholqr2_status"] = np.array(status)
out["cond_svqb2_rank"] = np.array(ranks)

# plans
out["default_tsqr_panel_rows"] = np.array([ref.default_tsqr_plan(10**6, n)[1] for n in (1, 8, 16, 32, 64)])
out["default_gram_panel_rows"] = np.array([ref.default_gram_plan(10**6, n)[1] for n in (1, 8, 16, 32, 64, 200)])
out["block_ranges_m1003_k7_b16"] = np.array([ref.block_range(1003, 7, 16, i) for i in range(7)])

dst = Path(__file__).with_name("reference_vectors.npz")
np.savez_compressed(dst, **out)
print(f"wrote {dst} ({dst.stat().st_size / 1024:.1f} KiB, {len(out)} arrays)")
