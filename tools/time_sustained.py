"""Burst and sustained (after 300 ms of back-to-back calls) TSQR throughput per kernel family.
python tools/time_sustained.py n1,n2,... kind1,kind2,... [LOG2_ROWS]"""
import sys
import time
from pathlib import Path

import os
sys.path.insert(0, os.environ.get("SQB_PKG_ROOT", str(Path(__file__).resolve().parents[1])))  # A/B: another build
import torch  # noqa: E402
import paper_2603_20889_b200 as sq  # noqa: E402

ns = [int(v) for v in sys.argv[1].split(",")]
kinds = sys.argv[2].split(",")
log2m = int(sys.argv[3]) if len(sys.argv) > 3 else 27
ctx = sq.Context(0)
ctx.use_torch_stream()


def timed(fn, reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for n in ns:
    m = 1 << log2m
    x = ctx.fill_gaussian(m, n, seed=1234)
    for rnd in range(2):
        for kind in kinds:
            ctx.set_tsqr_kernel(kind)
            fn = lambda: ctx.tsqr_qless(x)
            for _ in range(3):
                fn()
            torch.cuda.synchronize()
            time.sleep(1.0)
            burst = timed(fn, 20)
            t_end = time.perf_counter() + 0.3
            while time.perf_counter() < t_end:
                for _ in range(8):
                    fn()
                torch.cuda.synchronize()
            sust = timed(fn, 50)
            gb = 8.0 * m * n / 1e6
            print(f"n={n:2d} {kind:6s} burst {gb / burst:7.1f} GB/s   sustained {gb / sust:7.1f} GB/s", flush=True)
    del x
    torch.cuda.empty_cache()
