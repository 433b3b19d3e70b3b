"""Quick device-side timing of one method over a list of column counts.
python tools/time_methods.py METHOD n1,n2,... [LOG2_ELEMS] [REPS] [KERNEL]   (m = 2^LOG2_ELEMS / n rows;
KERNEL = auto | thread | fold | mma forces a TSQR kernel family)"""
import os
import sys
from pathlib import Path

sys.path.insert(0, os.environ.get("SQB_PKG_ROOT", str(Path(__file__).resolve().parents[1])))  # A/B: an older build
import torch  # noqa: E402
import paper_2603_20889_b200 as sq  # noqa: E402

method = sys.argv[1]
ns = [int(v) for v in sys.argv[2].split(",")]
log2e = int(sys.argv[3]) if len(sys.argv) > 3 else 29
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 5
ctx = sq.Context(0)
ctx.use_torch_stream()
if len(sys.argv) > 5:
    ctx.set_tsqr_kernel(sys.argv[5])
for n in ns:
    m = (1 << log2e) // n
    m -= m % 2
    x = ctx.fill_gaussian(m, n, seed=1234)
    if method in ("tsmRttsmR", "tsmmttsmm"):  # the second-pass kernels alone, factor = R of the matrix itself
        r = ctx.cholqr2(x)
        fn = (lambda xx: ctx.tsmRttsmR(xx, r)) if method == "tsmRttsmR" else (lambda xx: ctx.tsmmttsmm(xx, r))
    else:
        fn = {"tsqr": ctx.tsqr_qless, "stage1": ctx.tsqr_stage1, "tsmttsm": ctx.tsmttsm,
              "cholqr2": ctx.cholqr2, "svqb2": ctx.svqb2}[method]
    for _ in range(2):
        fn(x)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn(x)
    e1.record()
    torch.cuda.synchronize()
    ctx.synchronize()
    ms = e0.elapsed_time(e1) / reps
    gbs = 8.0 * m * n / ms / 1e6
    print(f"{method} n={n:3d} m={m:10d} {ms:9.3f} ms {gbs:8.1f} GB/s  {2.0*m*n*n/ms/1e9:6.2f} TF(2mn^2)", flush=True)
    del x
    torch.cuda.empty_cache()
