"""N > 1 host logic on CPU: two gloo ranks, row slabs, all-gather of triangles / all-reduce of Gram
matrices through paper_2603_20889_b200.sharding.  The per-slab kernels are stood in for by the CPU
oracle (test infrastructure); what is under test is the exchange and the combine wiring."""
import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, m, n, out_dir):
    import torch
    import torch.distributed as dist
    sys.path.insert(0, str(ROOT))
    sys.path.insert(0, str(ROOT / "tests"))
    import oracle
    from paper_2603_20889_b200 import sharding

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    x = oracle.gaussian(m, n, 99)
    lo, hi = sharding.slab_bounds(m, world, rank)
    xl = torch.from_numpy(np.ascontiguousarray(x[lo:hi]))

    def to_np(t):
        return np.asfortranarray(t.numpy())

    def local_qr(t):
        if t.shape[0] == 0:
            return torch.zeros((n, n), dtype=torch.float64)
        return torch.from_numpy(np.ascontiguousarray(oracle.port.block_qless_qr(to_np(t), 64)))

    def stack_qr(y):
        yy = to_np(y)
        return torch.from_numpy(np.ascontiguousarray(oracle.port.tsqr_qless(yy, 1, yy.shape[0])))

    r = sharding.tsqr_qless_sharded(xl, local_qr, stack_qr, dist)
    rc = sharding.cholqr2_sharded(
        xl,
        lambda t: torch.from_numpy(np.ascontiguousarray(oracle.port.tsmttsm(to_np(t), 1, 64))),
        lambda t, r1: torch.from_numpy(np.ascontiguousarray(oracle.port.tsmRttsmR(to_np(t), to_np(r1), 1, 64))),
        lambda c: torch.from_numpy(np.ascontiguousarray(oracle.port.cholesky(to_np(c)))),
        lambda a, b: torch.from_numpy(np.ascontiguousarray(oracle.port.triangular_multiply(to_np(a), to_np(b)))),
        dist)
    np.save(Path(out_dir) / f"r_{rank}.npy", r.numpy())
    np.save(Path(out_dir) / f"rc_{rank}.npy", rc.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("m,n", [(4001, 6), (5, 3)])
def test_two_rank_combine_matches_single_process(tmp_path, m, n):
    import torch.multiprocessing as mp
    import oracle

    port = _free_port()
    mp.spawn(_worker, args=(2, port, m, n, str(tmp_path)), nprocs=2, join=True)
    x = oracle.gaussian(m, n, 99)
    r_ref = oracle.port.reference_hhqr(x)
    bound = 64 * n * np.finfo(np.float64).eps * np.linalg.norm(x)
    r0, r1 = np.load(tmp_path / "r_0.npy"), np.load(tmp_path / "r_1.npy")
    assert np.array_equal(r0, r1)  # every rank ends with the same R
    assert np.linalg.norm(r0 - r_ref) <= bound
    rc0, rc1 = np.load(tmp_path / "rc_0.npy"), np.load(tmp_path / "rc_1.npy")
    assert np.array_equal(rc0, rc1)
    assert np.linalg.norm(rc0 - r_ref) <= bound
