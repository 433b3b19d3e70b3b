"""Times the n x n device kernels (Cholesky, Jacobi eigensolver, svqb_pass): python tools/time_small.py"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
import paper_2603_20889_b200 as sq

ctx = sq.Context(0)
ctx.use_torch_stream()
for n in (8, 16, 32, 48, 64):
    a = np.random.default_rng(n).standard_normal((4 * n, n))
    c = torch.from_numpy(np.ascontiguousarray((a.T @ a).T)).cuda().t()
    vals = ctx.empty_matrix(n, 1)
    def t(fn, reps=20):
        fn(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record(); torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps * 1e3
    I64 = sq.I64
    vecs = ctx.empty_matrix(n, n)
    def eig():
        ctx._check(ctx.lib.sqb_eigh_small_dev(ctx.handle, ctx._ptr(c), I64(n), ctx._ptr(vals), ctx._ptr(vecs)), "eigh")
    print(f"n={n:3d} cholesky {t(lambda: ctx.cholesky(c)):8.1f} us   eigh {t(eig):9.1f} us", flush=True)
