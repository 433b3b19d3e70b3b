"""Runs the BASELINE.json configurations other than the column sweep (which bench.py owns) on one
B200 and writes gpurun_out/configs_<tag>.json:

  C1  1,000,000 x 8 Gaussian: TSQR / CholQR2 / SVQB2 vs the compiled CPU reference (R parity, times)
  C3  4e7 x 32 with cond 1e2..1e12 (device-side restatement of the reference generator):
      TSQR stability vs CholQR2 / SVQB2 failure, R error vs the reference, orthogonality loss
      measured with the fused (X R^-1)^T (X R^-1) kernel (Q is never written)
  C4  least squares via Q-less QR of [A b], 1e9 x 16 on ONE GPU (128 GB resident), checked against
      the planted solution and across methods

python tools/run_configs.py [tag] [--small]
"""
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import oracle  # noqa: E402  (test infrastructure: the checker, never the thing measured)
import paper_2603_20889_b200 as sq  # noqa: E402

tag = next((a for a in sys.argv[1:] if not a.startswith("--")), "r01")
small = "--small" in sys.argv
EPS = np.finfo(np.float64).eps
ctx = sq.Context(0)
ctx.use_torch_stream()
ref = oracle.ref or oracle.port
out = {"device": torch.cuda.get_device_name(0), "host_threads": getattr(ref, "threads", 1)}


def gpu_ms(fn, reps=5, warm=2):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    ctx.synchronize()
    return e0.elapsed_time(e1) / reps


def cpu_s(fn, reps=3):
    fn()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return min(ts)


# ---- C1 ----------------------------------------------------------------------------------------
m, n = 1_000_000, 8
x = ctx.fill_gaussian(m, n, seed=1234)
xh = np.asfortranarray(x.cpu().numpy())
c1 = {"m": m, "n": n}
r_ref = ref.tsqr_qless(xh)
r_hh = oracle.port.reference_hhqr(xh)
bound = 64 * n * EPS * np.linalg.norm(xh)
for meth, fn, cfn in (("tsqr", ctx.tsqr_qless, ref.tsqr_qless), ("cholqr2", ctx.cholqr2, ref.cholqr2)):
    r = fn(x)
    ctx.synchronize()
    r = r.cpu().numpy()
    c1[meth] = {"gpu_ms_resident": gpu_ms(lambda: fn(x), 20, 3),
                "gpu_ms_host_api": 1e3 * cpu_s(lambda: fn(xh)),
                "cpu_reference_ms": 1e3 * cpu_s(lambda: cfn(xh)),
                "err_vs_reference_tsqr": float(np.linalg.norm(r - r_ref)),
                "err_vs_reference_hhqr": float(np.linalg.norm(r - r_hh)), "bound": float(bound)}
tr, z, sg, rank = ctx.svqb2(x)
ctx.synchronize()
c1["svqb2"] = {"gpu_ms_resident": gpu_ms(lambda: ctx.svqb2(x), 20, 3), "rank": int(rank.item()),
               "cpu_reference_ms": 1e3 * cpu_s(lambda: ref.svqb2(xh)),
               "sigma_rel_err": float(np.linalg.norm(sg.cpu().numpy() - np.linalg.svd(xh, compute_uv=False))
                                      / np.linalg.norm(xh, 2))}
out["C1"] = c1
del x
print("C1 done", json.dumps(c1)[:300], flush=True)

# ---- C3 ----------------------------------------------------------------------------------------
m, n = (4_000_000 if small else 40_000_000), 32
rows = []
x = ctx.empty_matrix(m, n)
for kappa in (1e2, 1e4, 1e6, 1e8, 1e10, 1e12):
    ctx.generate(m, n, kappa, seed=42, out=x)
    ctx.synchronize()
    row = {"kappa": kappa, "m": m, "n": n}
    r = ctx.tsqr_qless(x)
    ctx.synchronize()
    row["tsqr_ms"] = gpu_ms(lambda: ctx.tsqr_qless(x), 3, 1)
    # orthogonality of Q = X R^-1 without writing Q: |(X R^-1)^T (X R^-1) - I|_2
    c2 = ctx.tsmRttsmR(x, r)
    ctx.synchronize()
    row["tsqr_orth_loss_2norm"] = float(np.linalg.norm(c2.cpu().numpy() - np.eye(n), 2))
    xh = np.asfortranarray(x.cpu().numpy())
    xn = float(np.linalg.norm(xh))
    t0 = time.perf_counter()
    r_cpu = ref.tsqr_qless(xh)
    row["cpu_reference_tsqr_s"] = time.perf_counter() - t0
    row["tsqr_err_vs_reference"] = float(np.linalg.norm(r.cpu().numpy() - r_cpu))
    row["bound_64_n_eps_normX"] = 64 * n * EPS * xn
    for meth, fn in (("cholqr2", ctx.cholqr2), ("svqb2", ctx.svqb2)):
        try:
            res = fn(x)
            ctx.synchronize(meth)
            row[meth + "_ms"] = gpu_ms(lambda: fn(x), 3, 1)
            if meth == "cholqr2":
                rc = res.cpu().numpy()
                row["cholqr2_err_vs_tsqr"] = float(np.linalg.norm(rc - r.cpu().numpy()))
                c2 = ctx.tsmRttsmR(x, res)
                ctx.synchronize()
                row["cholqr2_orth_loss_2norm"] = float(np.linalg.norm(c2.cpu().numpy() - np.eye(n), 2))
            else:
                row["svqb2_rank"] = int(res[3].item())
        except sq.Error as exc:
            row[meth] = type(exc).__name__ + (f"(pivot {exc.pivot_index})" if hasattr(exc, "pivot_index") else "")
    try:
        ref.cholqr2(xh)
        row["cpu_reference_cholqr2"] = "ok"
    except oracle.OracleError as exc:
        row["cpu_reference_cholqr2"] = f"{exc.kind}(pivot {exc.index})"
    row["cpu_reference_svqb2_rank"] = ref.svqb2(xh)[3]
    rows.append(row)
    print("C3", json.dumps(row), flush=True)
    del xh
out["C3"] = rows
del x
torch.cuda.empty_cache()

# ---- C4 ----------------------------------------------------------------------------------------
m, n = (50_000_000 if small else 1_000_000_000), 15
a = ctx.fill_gaussian(m, n, seed=77)
x_true = torch.arange(1, n + 1, dtype=torch.float64, device="cuda") / n
rhs = ctx.fill_gaussian(m, 1, seed=78)[:, 0].contiguous()
rhs.mul_(0.01)
for j in range(n):  # rhs += A[:, j] * x_true[j], column by column (harness arithmetic only)
    rhs.add_(a[:, j], alpha=float(x_true[j]))
torch.cuda.synchronize()
c4 = {"m": m, "n_A": n, "cols_streamed": n + 1, "bytes": 8.0 * m * (n + 1)}
sols = {}
for meth in ("tsqr", "cholqr2"):
    xs, res = ctx.solve_lstsq(a, rhs, meth)
    ctx.synchronize()
    ms = gpu_ms(lambda: ctx.solve_lstsq(a, rhs, meth), 3, 1)
    sols[meth] = xs.cpu().numpy()
    c4[meth] = {"ms": ms, "gbs": 8.0 * m * (n + 1) / ms / 1e6,
                "max_abs_err_vs_planted": float(np.abs(sols[meth] - x_true.cpu().numpy()).max()),
                "residual_norm": float(res.item()), "expected_residual": 0.01 * np.sqrt(m - n)}
c4["tsqr_vs_cholqr2_max_abs_diff"] = float(np.abs(sols["tsqr"] - sols["cholqr2"]).max())
mc = 10_000_000
ah = np.asfortranarray(a[:mc].cpu().numpy())
bh = rhs[:mc].cpu().numpy()
xs_gpu, _ = ctx.solve_lstsq(a[:mc], rhs[:mc].contiguous(), "tsqr")
ctx.synchronize()
xs_cpu, _ = ref.solve_lstsq(ah, bh, "tsqr")
c4["parity_vs_cpu_reference_at_1e7_rows"] = float(np.abs(xs_gpu.cpu().numpy() - xs_cpu).max())
out["C4"] = c4
print("C4", json.dumps(c4), flush=True)

del a, rhs
torch.cuda.empty_cache()

# ---- C5 ----------------------------------------------------------------------------------------
# transitional regime: the Gram matrix of a 2^24 x n matrix, n = 128 / 256, on the FP64 tensor cores.
# CholQR2 and SVQB2 run up to 128 columns (fused solve / multiply + Gram on the tensor cores).
# The reference's tsqr_qless rejects n > 64 (tsqr.cpp:188), so there is no TSQR arm at these widths;
# the widest TSQR (n = 64) is timed beside it for the flop-rate comparison.
m = (1 << 20) if small else (1 << 24)
c5 = []
for n in (64, 128, 256):
    x = ctx.fill_gaussian(m, n, seed=1234)
    row = {"m": m, "n": n}
    ms = gpu_ms(lambda: ctx.tsmttsm(x), 5, 2)
    tiles = (n + 7) // 8 if n <= 64 else 16 * ((n + 127) // 128)
    pairs = tiles * (tiles + 1) // 2
    row["tsmttsm_ms"] = ms
    row["gbs"] = 8.0 * m * n / ms / 1e6
    row["nominal_tflops_2mn2"] = 2.0 * m * n * n / ms / 1e9
    row["executed_dmma_tflops"] = 2.0 * m * pairs * 64 / ms / 1e9
    row["dmma_pipe_util_vs_37.1"] = row["executed_dmma_tflops"] / 37.1
    mc = 1 << 17
    xh = np.asfortranarray(x[:mc].cpu().numpy())
    c_gpu = ctx.tsmttsm(x[:mc])
    ctx.synchronize()
    c_ref = ref.tsmttsm(xh)
    row["parity_err_F_at_2^17_rows"] = float(np.linalg.norm(c_gpu.cpu().numpy() - c_ref))
    row["parity_bound_5_n_eps_normX2"] = float(5 * n * EPS * np.linalg.norm(xh) ** 2)
    if n <= 256:  # CholQR2 (n <= 256) / SVQB2 (n <= 128, eigh_small's limit), parity against the reference
        row["cholqr2_ms"] = gpu_ms(lambda: ctx.cholqr2(x), 3, 1)
        row["cholqr2_gbs_effective"] = 8.0 * m * n / row["cholqr2_ms"] / 1e6
        row["cholqr2_second_sweep_useful_tflops_2mn2"] = 2.0 * m * n * n / (row["cholqr2_ms"] - ms) / 1e9
        if n <= 128:
            row["svqb2_ms"] = gpu_ms(lambda: ctx.svqb2(x), 3, 1)
            row["svqb2_gbs_effective"] = 8.0 * m * n / row["svqb2_ms"] / 1e6
        r_gpu = ctx.cholqr2(x[:mc])
        ctx.synchronize()
        r_ref = ref.cholqr2(xh)
        row["cholqr2_parity_err_F_at_2^17_rows"] = float(np.linalg.norm(r_gpu.cpu().numpy() - r_ref))
        row["cholqr2_parity_bound_64_n_eps_normX"] = float(64 * n * EPS * np.linalg.norm(xh))
    if n <= 64:
        row["tsqr_ms"] = gpu_ms(lambda: ctx.tsqr_qless(x), 3, 1)
        row["tsqr_tflops_2mn2"] = 2.0 * m * n * n / row["tsqr_ms"] / 1e9
    c5.append(row)
    print("C5", json.dumps(row), flush=True)
    del x
    torch.cuda.empty_cache()
out["C5"] = c5

dst = ROOT / "gpurun_out" / f"configs_{tag}.json"
dst.parent.mkdir(exist_ok=True)
dst.write_text(json.dumps(out, indent=1))
print("wrote", dst)
