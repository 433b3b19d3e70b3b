"""The library's multi-GPU protocol at world > 1 on ONE GPU.

Two routes, both through the C ABI:
 * the exported halves - sqb_tsqr_local_dev per slab, sqb_tsqr_combine_dev / sqb_gram_combine_dev
   over world in {2, 4, 8} gathered blocks - in a single process;
 * the sharded drivers themselves (sqb_{tsqr_qless,cholqr2,svqb2,solve_lstsq}_sharded_dev) in
   2 and 4 processes that share cuda:0, with the n x n all-gather served by torch.distributed/gloo
   through the library's exchange hook (sharding.attach(..., transport="torch")) - the same driver
   code that runs over NCCL on a multi-GPU box (NCCL refuses two ranks on one device).
Oracle: the compiled reference (oracle.ref) where built, else the C port."""
import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest

from conftest import EPS, r_bound

ROOT = Path(__file__).resolve().parents[1]
pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world", [2, 4, 8])
@pytest.mark.parametrize("m,n", [(30011, 8), (9001, 16), (20000, 33), (5000, 64), (11, 5)])
def test_combine_abi_matches_full_matrix(ctx, oracle, world, m, n):
    import torch
    from paper_2603_20889_b200 import sharding
    best = oracle.ref or oracle.port
    x = ctx.fill_gaussian(m, n, seed=77)
    xh = np.asfortranarray(x.cpu().numpy())
    tris, grams = [], []
    for g in range(world):
        lo, hi = sharding.slab_bounds(m, world, g)
        slab = x[lo:hi] if hi > lo else ctx.empty_matrix(0, n)   # row slab of the column-major matrix (ld = m)
        tris.append(ctx.tsqr_local(slab))
        grams.append(ctx.tsmttsm(slab) if hi > lo else torch.zeros_like(tris[-1]))
    r = ctx.tsqr_combine(tris)
    c = ctx.gram_combine(grams)
    r_full = ctx.tsqr_qless(x)
    ctx.synchronize()
    rh = r.cpu().numpy()
    assert np.all(np.tril(rh, -1) == 0.0) and np.all(np.diag(rh) >= 0.0)
    assert np.linalg.norm(rh - best.tsqr_qless(xh)) <= r_bound(xh)
    assert np.linalg.norm(rh - oracle.port.reference_hhqr(xh)) <= r_bound(xh)
    assert np.linalg.norm(rh - r_full.cpu().numpy()) <= r_bound(xh)
    # ascending-rank sum of the partial Grams: exactly the sequential sum, and the reference's C
    seq = grams[0].cpu().numpy().copy()
    for gpart in grams[1:]:
        seq += gpart.cpu().numpy()
    assert np.array_equal(c.cpu().numpy(), seq)
    assert np.linalg.norm(c.cpu().numpy() - best.tsmttsm(xh)) <= 5 * n * EPS * np.linalg.norm(xh) ** 2


def _worker(rank, world, port, m, n, out_dir):
    import torch
    import torch.distributed as dist
    sys.path.insert(0, str(ROOT))
    import paper_2603_20889_b200 as sq
    from paper_2603_20889_b200 import sharding

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    ctx = sq.Context(0)
    ctx.use_torch_stream()
    assert sharding.attach(ctx, dist, transport="torch") == "torch"
    lo, hi = sharding.slab_bounds(m, world, rank)
    # every rank generates its own rows of ONE logical m x (n+1) Gaussian matrix [A rhs]
    xl = ctx.fill_gaussian(hi - lo, n + 1, seed=4321, row_offset=lo, m_total=m)
    a, rhs = xl[:, :n], xl[:, n].contiguous()
    r = ctx.tsqr_qless_sharded(a)
    rc = ctx.cholqr2_sharded(a)
    tr, z, sg, rk = ctx.svqb2_sharded(a)
    xs, res = ctx.solve_lstsq_sharded(a, rhs)
    ctx.synchronize("sharded")
    assert ctx.exchange.calls == 1 + 2 + 2 + 1  # one all-gather per TSQR, two per Gram method
    np.savez(Path(out_dir) / f"rank{rank}.npz", r=r.cpu().numpy(), rc=rc.cpu().numpy(), z=z.cpu().numpy(),
             tr=tr.cpu().numpy(), sg=sg.cpu().numpy(), rk=rk.cpu().numpy(), xs=xs.cpu().numpy(),
             res=res.cpu().numpy(), xl=xl.cpu().numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,m,n", [(2, 40001, 8), (4, 50000, 16), (4, 9, 3), (2, 30000, 40)])
def test_sharded_drivers_multi_process_one_gpu(tmp_path, oracle, world, m, n):
    import torch.multiprocessing as mp
    best = oracle.ref or oracle.port
    port = _free_port()
    mp.spawn(_worker, args=(world, port, m, n, str(tmp_path)), nprocs=world, join=True)
    outs = [np.load(tmp_path / f"rank{g}.npz") for g in range(world)]
    xfull = np.asfortranarray(np.concatenate([o["xl"] for o in outs], axis=0))
    assert xfull.shape == (m, n + 1)
    a, rhs = np.asfortranarray(xfull[:, :n]), np.ascontiguousarray(xfull[:, n])
    for key in ("r", "rc", "z", "tr", "sg", "rk", "xs", "res"):  # every rank ends with the same bits
        for o in outs[1:]:
            assert np.array_equal(outs[0][key], o[key]), key
    o = outs[0]
    bound = r_bound(a)
    r_ref = best.tsqr_qless(a)
    assert np.linalg.norm(o["r"] - r_ref) <= bound
    assert np.linalg.norm(o["rc"] - best.cholqr2(a)) <= bound
    assert np.linalg.norm(o["rc"] - r_ref) <= bound
    # SVQB2: Z^T Z = X^T X, Z B = I, full rank (bases are not unique: parity on invariants)
    c = a.T @ a
    assert int(o["rk"][0]) == n
    assert np.linalg.norm(o["z"].T @ o["z"] - c) <= 50 * n * EPS * np.linalg.norm(a) ** 2
    assert np.linalg.norm(o["z"] @ o["tr"] - np.eye(n)) <= 1e-10
    xs_ref, res_ref = best.solve_lstsq(a, rhs, "tsqr")
    assert np.allclose(o["xs"], xs_ref, rtol=1e-9, atol=1e-12)
    assert abs(float(o["res"][0]) - res_ref) <= 1e-10 * max(res_ref, 1.0)


@pytest.mark.gpu
@pytest.mark.parametrize("extra", [["--m", "2097152", "--no-cpu"], ["--config", "c4", "--c4-rows", "4000000"]])
def test_bench_multi_rank_flow_on_one_gpu(extra):
    """`bench.py --gpus 2` end to end - it starts its own ranks, every rank runs the sharded drivers, rank 0
    prints exactly one JSON line with n_gpus = 2 - with both ranks on cuda:0 over gloo (`--share-gpu`: NCCL
    refuses two ranks on one device).  A flow check of the launcher path, not a scaling number."""
    import json
    import subprocess
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    out = subprocess.run([sys.executable, str(root / "bench.py"), "--gpus", "2", "--share-gpu", "--steps", "3",
                          "--warmup", "3", "--no-sweep"] + extra, capture_output=True, text=True, cwd=root, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.strip()]
    assert len(lines) == 1, out.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["gpu_launches"] > 0
    assert "flow check" in d["config"]["transport"]
