import sys, numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import paper_2603_20889_b200 as sq
from conftest import gaussian
ctx = sq.default_context(0)
bad = 0
for it in range(int(sys.argv[1])):
    for (m, n) in [(5000, 64), (6000, 48), (10000, 32)]:
        x = gaussian(m, n, seed=7 * n + it)
        bm = gaussian(n, n, seed=99) / np.sqrt(m)
        c3 = ctx.tsmmttsmm(x, bm)
        ref = (x @ bm).T @ (x @ bm)
        e = np.linalg.norm(c3 - ref) / np.linalg.norm(ref)
        r1 = np.linalg.cholesky(x.T @ x).T.copy(order="F")
        c2 = ctx.tsmRttsmR(x, r1)
        e2 = np.linalg.norm(c2 - np.eye(n))
        c1 = ctx.tsmttsm(x)
        e1 = np.linalg.norm(c1 - x.T @ x) / np.linalg.norm(ref)
        if not (e < 1e-12 and e2 < 1e-10 and e1 < 1e-10):
            bad += 1
            print("BAD", it, m, n, e, e2, e1, flush=True)
print("bad", bad)
