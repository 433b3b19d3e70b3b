"""Device-side timing of the n x n solves (one CTA each) on the Gram matrix of a Gaussian X.
python tools/time_small.py n1,n2,... [REPS]      prints ms per call of cholesky / eigh_small / svqb_pass"""
import ctypes as C
import os
import sys
from pathlib import Path

sys.path.insert(0, os.environ.get("SQB_PKG_ROOT", str(Path(__file__).resolve().parents[1])))  # A/B: an older build
import torch  # noqa: E402
import paper_2603_20889_b200 as sq  # noqa: E402

ns = [int(v) for v in sys.argv[1].split(",")]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
ctx = sq.Context(0)
ctx.use_torch_stream()
I64 = C.c_int64


def timed(fn):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for n in ns:
    x = ctx.fill_gaussian(1 << 16, n, seed=77)
    c = ctx.tsmttsm(x)
    out = [ctx.empty_matrix(n, n) for _ in range(3)]
    vals = torch.empty(n, dtype=torch.float64, device=c.device)
    rank = torch.zeros(1, dtype=torch.int64, device=c.device)
    p = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
    row = [f"n={n:3d}"]
    if n <= 256:
        row.append("cholesky %7.3f ms" % timed(lambda: ctx.lib.sqb_cholesky_dev(ctx.handle, p(c), I64(n), p(out[0]))))
    if n <= 128:
        row.append("eigh %7.3f ms" % timed(
            lambda: ctx.lib.sqb_eigh_small_dev(ctx.handle, p(c), I64(n), p(vals), p(out[0]))))
        row.append("svqb_pass %7.3f ms" % timed(
            lambda: ctx.lib.sqb_svqb_pass_dev(ctx.handle, p(c), I64(n), p(out[1]), p(out[2]), p(vals), p(rank))))
    ctx.synchronize()
    print("  ".join(row), flush=True)
