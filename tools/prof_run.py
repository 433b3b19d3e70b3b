"""Tiny driver for ncu captures: python tools/prof_run.py METHOD N [LOG2_M] [REPS]
METHOD in {tsqr, stage1, tsmttsm, cholqr2, svqb2}."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402
import paper_2603_20889_b200 as sq  # noqa: E402

method, n = sys.argv[1], int(sys.argv[2])
m = 1 << (int(sys.argv[3]) if len(sys.argv) > 3 else 25)
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 2
ctx = sq.Context(0)
ctx.use_torch_stream()
x = ctx.fill_gaussian(m, n, seed=1234)
fn = {"tsqr": ctx.tsqr_qless, "stage1": ctx.tsqr_stage1, "tsmttsm": ctx.tsmttsm, "cholqr2": ctx.cholqr2,
      "svqb2": ctx.svqb2}[method]
for _ in range(reps):
    fn(x)
ctx.synchronize()
print("done", method, n, m)
