"""skinny-qr style command line (reference SPEC.md "bench-driver" external interface; the reference
itself ships no CLI):

  python -m paper_2603_20889_b200 bench --mn-product P --cols 1,8,16,32,64 --methods tsqr,cholqr2,svqb2
         [--kappa K] [--seed S] [--reps 50] [--warmups 3] [--hw B200] [--out results.csv] [--format csv|json|text]
  python -m paper_2603_20889_b200 lstsq --matrix A.tskm --rhs b.tskm [--method tsqr|cholqr2]
  python -m paper_2603_20889_b200 qr    --matrix A.tskm [--method tsqr|cholqr2] [--out R.tskm]
  python -m paper_2603_20889_b200 model --hw B200 --kernel tsqr --m M --n N

`model` is pure arithmetic; everything else needs the CUDA library and an sm_100 device (no CPU fallback).
Exit code 0 iff every accuracy residual passes its threshold (orthogonality and Gram consistency
<= 1e-12 * max(1, kappa-dependent slack), as in SPEC.md acceptance criterion 5).
"""
from __future__ import annotations

import argparse
import csv
import io as _io
import json
import sys

COLUMNS = ["method", "m", "n", "kappa", "seed", "reps", "t_mean_s", "t_min_s", "orth_resid", "gram_resid",
           "large_reads", "flops", "model_time_s", "model_ratio"]


def render(rows, fmt):
    if fmt == "json":
        return json.dumps(rows, indent=1) + "\n"
    if fmt == "text":
        lines = ["  ".join(f"{c:>14s}" for c in COLUMNS)]
        for r in rows:
            lines.append("  ".join(f"{r[c]:>14.6g}" if isinstance(r[c], float) else f"{str(r[c]):>14s}" for c in COLUMNS))
        return "\n".join(lines) + "\n"
    buf = _io.StringIO()
    w = csv.DictWriter(buf, fieldnames=COLUMNS)
    w.writeheader()
    for r in rows:
        w.writerow(r)
    return buf.getvalue()


def cmd_model(a):
    from . import perf_model as pm
    hw = pm.find_hardware(a.hw) or pm.load_hardware_spec(a.hw)
    t = pm.composite_time(hw, a.kernel, a.m, a.n) if a.kernel in pm.METHODS and a.kernel not in pm.KERNELS \
        else pm.predict_time(hw, a.kernel, a.m, a.n)
    print(json.dumps({"hw": hw.name, "kernel": a.kernel, "m": a.m, "n": a.n, "machine_balance": pm.machine_balance(hw),
                      "time_s": t}))
    return 0


def cmd_bench(a):
    import numpy as np
    import torch
    import paper_2603_20889_b200 as sq
    from . import perf_model as pm
    if a.reps < 1:
        raise sq.ArgumentError("bench: reps must be >= 1")
    hw = pm.find_hardware(a.hw) or pm.load_hardware_spec(a.hw)
    ctx = sq.Context(0)
    ctx.use_torch_stream()
    rows, ok = [], True
    for n in [int(v) for v in a.cols.split(",")]:
        m = max(n, round(a.mn_product / n))
        x = ctx.generate(m, n, a.kappa, seed=a.seed) if a.kappa > 1.0 else ctx.fill_gaussian(m, n, seed=a.seed)
        xnorm2 = float(torch.linalg.matrix_norm(x) ** 2)
        for method in a.methods.split(","):
            row = {c: "" for c in COLUMNS}
            row.update(method=method, m=m, n=n, kappa=a.kappa, seed=a.seed, reps=a.reps)
            try:
                fn = {"tsqr": ctx.tsqr_qless, "cholqr2": ctx.cholqr2, "svqb2": ctx.svqb2}[method]
                for _ in range(a.warmups):
                    fn(x)
                torch.cuda.synchronize()
                ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(a.reps)]
                for e0, e1 in ev:
                    e0.record()
                    res = fn(x)
                    e1.record()
                torch.cuda.synchronize()
                ctx.synchronize(method)
                ts = [e0.elapsed_time(e1) * 1e-3 for e0, e1 in ev]
                # residuals without writing Q: |(X R^-1)^T (X R^-1) - I|_2 and |R^T R - X^T X|_F / |X|_F^2
                if method == "svqb2":
                    bmat = res[0]
                    g = ctx.tsmmttsmm(x, bmat)
                    rank = int(res[3].item())
                    eye = np.zeros((n, n))
                    eye[:rank, :rank] = np.eye(rank)
                    orth = float(np.linalg.norm(g.cpu().numpy() - eye, 2))
                    gram = float("nan")
                else:
                    g = ctx.tsmRttsmR(x, res)
                    c = ctx.tsmttsm(x)
                    ctx.synchronize()
                    rr = res.cpu().numpy()
                    orth = float(np.linalg.norm(g.cpu().numpy() - np.eye(n), 2))
                    gram = float(np.linalg.norm(rr.T @ rr - c.cpu().numpy()) / xnorm2)
                passes = 1 if method == "tsqr" else 2
                kern = {"tsqr": "tsqr", "cholqr2": "tsmRttsmR", "svqb2": "tsmmttsmm"}[method]
                flops = pm.kernel_flops(kern, m, n) + (pm.kernel_flops("tsmttsm", m, n) if passes == 2 else 0.0)
                model = pm.composite_time(hw, method, m, n)
                row.update(t_mean_s=sum(ts) / len(ts), t_min_s=min(ts), orth_resid=orth, gram_resid=gram,
                           large_reads=passes * m * n, flops=flops, model_time_s=model, model_ratio=(sum(ts) / len(ts)) / model)
                tol = 1e-12 * max(1.0, a.kappa if method == "tsqr" else a.kappa ** 2)
                ok = ok and orth <= tol
            except sq.Error as exc:  # per-row report, the grid continues
                row["orth_resid"] = type(exc).__name__
            rows.append(row)
        del x
        torch.cuda.empty_cache()
    text = render(rows, a.format)
    if a.out:
        with open(a.out, "w") as f:
            f.write(text)
    else:
        sys.stdout.write(text)
    return 0 if ok else 1


def cmd_lstsq(a):
    import paper_2603_20889_b200 as sq
    from . import io as tio
    ctx = sq.Context(0)
    ctx.use_torch_stream()
    amat = tio.matrix_read_device(a.matrix, ctx)
    rhs = tio.matrix_read_device(a.rhs, ctx)
    if rhs.shape[1] != 1 or rhs.shape[0] != amat.shape[0]:
        raise sq.DimensionError("lstsq: rhs must be an m x 1 matrix")
    xs, res = ctx.solve_lstsq(amat, rhs[:, 0].contiguous(), a.method)
    ctx.synchronize("lstsq")
    print(json.dumps({"x": xs.cpu().numpy().tolist(), "residual_norm": float(res.item())}))
    return 0


def cmd_qr(a):
    import paper_2603_20889_b200 as sq
    from . import io as tio
    ctx = sq.Context(0)
    ctx.use_torch_stream()
    x = tio.matrix_read_device(a.matrix, ctx)
    r = (ctx.tsqr_qless if a.method == "tsqr" else ctx.cholqr2)(x)
    ctx.synchronize("qr")
    rh = r.cpu().numpy()
    if a.out:
        tio.matrix_write(a.out, rh)
    else:
        print(json.dumps({"r": rh.tolist()}))
    return 0


def main(argv=None):
    ap = argparse.ArgumentParser(prog="python -m paper_2603_20889_b200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    b = sub.add_parser("bench")
    b.add_argument("--mn-product", type=float, default=float(1 << 23))
    b.add_argument("--cols", default="1,8,16,32,64")
    b.add_argument("--methods", default="tsqr,cholqr2,svqb2")
    b.add_argument("--kappa", type=float, default=1.0)
    b.add_argument("--seed", type=int, default=42)
    b.add_argument("--reps", type=int, default=50)
    b.add_argument("--warmups", type=int, default=3)
    b.add_argument("--hw", default="B200")
    b.add_argument("--out", default="")
    b.add_argument("--format", default="csv", choices=["csv", "json", "text"])
    b.set_defaults(fn=cmd_bench)
    l = sub.add_parser("lstsq")
    l.add_argument("--matrix", required=True)
    l.add_argument("--rhs", required=True)
    l.add_argument("--method", default="tsqr", choices=["tsqr", "cholqr2"])
    l.set_defaults(fn=cmd_lstsq)
    q = sub.add_parser("qr")
    q.add_argument("--matrix", required=True)
    q.add_argument("--method", default="tsqr", choices=["tsqr", "cholqr2"])
    q.add_argument("--out", default="")
    q.set_defaults(fn=cmd_qr)
    mo = sub.add_parser("model")
    mo.add_argument("--hw", default="B200")
    mo.add_argument("--kernel", required=True)
    mo.add_argument("--m", type=int, required=True)
    mo.add_argument("--n", type=int, required=True)
    mo.set_defaults(fn=cmd_model)
    a = ap.parse_args(argv)
    return a.fn(a)


if __name__ == "__main__":
    sys.exit(main())
