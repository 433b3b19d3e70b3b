"""Wide Gram (config 5) timing: python tools/time_gram_wide.py [LOG2_M]  -> ms, GB/s, executed DMMA TFLOP/s"""
import sys
from pathlib import Path
import os  # noqa: E402
sys.path.insert(0, os.environ.get("SQB_PKG_ROOT", str(Path(__file__).resolve().parents[1])))  # A/B: an older build
import torch  # noqa: E402
import paper_2603_20889_b200 as sq  # noqa: E402

log2m = int(sys.argv[1]) if len(sys.argv) > 1 else 24
ctx = sq.Context(0)
ctx.use_torch_stream()
for n in (96, 128, 192, 256):
    m = 1 << log2m
    x = ctx.fill_gaussian(m, n, seed=1234)
    for _ in range(2):
        ctx.tsmttsm(x)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    reps = 5
    for _ in range(reps):
        ctx.tsmttsm(x)
    e1.record()
    torch.cuda.synchronize()
    ctx.synchronize()
    ms = e0.elapsed_time(e1) / reps
    nt = 16 * ((n + 127) // 128)
    pairs = 136 if nt == 16 else 528
    print(f"tsmttsm n={n:3d} m=2^{log2m} {ms:8.3f} ms  {8.0*m*n/ms/1e6:8.1f} GB/s  nominal 2mn^2 {2.0*m*n*n/ms/1e9:6.2f} TF  "
          f"executed DMMA {2.0*m*pairs*64/ms/1e9:6.2f} TF", flush=True)
    if n > 128:  # CholQR2 through Q = X R^-1 per row slab + the wide SYRK (explicit Q slab, compute-bound regime)
        for _ in range(2):
            ctx.cholqr2(x)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(reps):
            ctx.cholqr2(x)
        e1.record()
        torch.cuda.synchronize()
        ctx.synchronize()
        ms2 = e0.elapsed_time(e1) / reps
        # second sweep: triangular GEMM m n^2 flops (executed at 8 x 8 tile granularity) + SYRK pairs
        nt2 = nt
        gemm_tiles = 16 * 17 // 2 + 16 * 16 + ((n - 128 + 7) // 8) * ((n - 128 + 7) // 8 + 1) // 2
        print(f"cholqr2 n={n:3d} m=2^{log2m} {ms2:8.3f} ms  {8.0*m*n/ms2/1e6:8.1f} GB/s effective  "
              f"second sweep {ms2-ms:8.3f} ms = useful {(2.0*m*n*n)/(ms2-ms)/1e9:6.2f} TF (m n^2 GEMM + m n^2 SYRK)", flush=True)
    if n <= 128:  # CholQR2 through the fused solve + Gram sweep (two reads of X)
        for _ in range(2):
            ctx.cholqr2(x)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(reps):
            ctx.cholqr2(x)
        e1.record()
        torch.cuda.synchronize()
        ctx.synchronize()
        ms2 = e0.elapsed_time(e1) / reps
        print(f"cholqr2 n={n:3d} m=2^{log2m} {ms2:8.3f} ms  {8.0*m*n/ms2/1e6:8.1f} GB/s effective  "
              f"second sweep {ms2-ms:8.3f} ms = executed DMMA {2.0*m*272*64/(ms2-ms)/1e9:6.2f} TF", flush=True)
        for _ in range(2):
            ctx.svqb2(x)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(reps):
            ctx.svqb2(x)
        e1.record()
        torch.cuda.synchronize()
        ctx.synchronize()
        ms3 = e0.elapsed_time(e1) / reps
        print(f"svqb2   n={n:3d} m=2^{log2m} {ms3:8.3f} ms  {8.0*m*n/ms3/1e6:8.1f} GB/s effective", flush=True)
    del x
    torch.cuda.empty_cache()
