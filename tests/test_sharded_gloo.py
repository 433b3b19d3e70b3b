"""N > 1 host logic on CPU: two gloo ranks driving paper_2603_20889_b200.sharding - the same
functions bench.py and the multi-rank GPU test use (slab_bounds, broadcast_bytes, max_over_ranks,
TorchExchange.gather_host).  The protocol itself lives in the C library (sqb_*_sharded_dev) and is
covered at world > 1 by tests/test_sharded_gpu.py; here its host side is replayed with the CPU oracle
standing in for the per-slab kernels (test infrastructure), in the library's order: local triangle ->
all-gather -> stack -> one more block QR; local Gram -> all-gather -> ascending-rank sum."""
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
    import torch.distributed as dist
    sys.path.insert(0, str(ROOT))
    sys.path.insert(0, str(ROOT / "tests"))
    import oracle
    from paper_2603_20889_b200 import sharding

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ex = sharding.TorchExchange(dist)
    assert (ex.rank, ex.world) == (rank, world)

    # launcher helpers
    uid = sharding.broadcast_bytes(bytes(range(128)) if rank == 0 else None, dist)
    assert uid == bytes(range(128))
    assert sharding.max_over_ranks(1.0 + rank, dist) == float(world)
    g = ex.gather_host(np.full(3, float(rank)))
    assert g.shape == (world, 3) and np.array_equal(g[:, 0], np.arange(world, dtype=np.float64))

    x = oracle.gaussian(m, n, 99)
    lo, hi = sharding.slab_bounds(m, world, rank)
    xl = np.asfortranarray(x[lo:hi])

    # TSQR: stage 2 with k = world (tsqr.cpp:175-195)
    r_local = oracle.port.block_qless_qr(xl, 64) if hi > lo else np.zeros((n, n), order="F")
    gathered = ex.gather_host(np.asfortranarray(r_local).ravel(order="F"))
    stack = np.asfortranarray(np.concatenate([blk.reshape(n, n, order="F") for blk in gathered], axis=0))
    r = oracle.port.tsqr_qless(stack, 1, stack.shape[0])

    # CholQR2: every Gram partial all-gathered and summed in ascending rank order (gram.cpp:81-92)
    def allsum(c):
        parts = ex.gather_host(np.asfortranarray(c).ravel(order="F"))
        acc = parts[0].copy()
        for blk in parts[1:]:
            acc += blk
        return np.asfortranarray(acc.reshape(n, n, order="F"))

    zero = np.zeros((n, n), order="F")
    r1 = oracle.port.cholesky(allsum(oracle.port.tsmttsm(xl, 1, 64) if hi > lo else zero))
    r2 = oracle.port.cholesky(allsum(oracle.port.tsmRttsmR(xl, r1, 1, 64) if hi > lo else zero))
    rc = oracle.port.triangular_multiply(r2, r1)
    np.save(Path(out_dir) / f"r_{rank}.npy", r)
    np.save(Path(out_dir) / f"rc_{rank}.npy", rc)
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


def test_slab_bounds_cover_rows_once():
    from paper_2603_20889_b200 import sharding
    for m, world in [(0, 3), (5, 8), (1000, 7), (2**27, 8), (10**9, 8)]:
        cuts = [sharding.slab_bounds(m, world, g) for g in range(world)]
        assert cuts[0][0] == 0 and cuts[-1][1] == m
        assert all(a[1] == b[0] for a, b in zip(cuts, cuts[1:]))
        assert all(lo <= hi for lo, hi in cuts)
    with pytest.raises(ValueError):
        sharding.slab_bounds(10, 2, 2)


def test_bench_spawn_command():
    """bench.py --gpus N (no torchrun around it) re-executes itself under torch.distributed.run."""
    sys.path.insert(0, str(ROOT))
    import bench
    import json
    import os
    argv = ["--gpus", "4", "--steps", "5", "--m", "1024", "--n", "8"]
    cmd = bench.spawn_command(4, argv, port=29999)
    assert cmd[1:4] == ["-m", "torch.distributed.run", "--nnodes=1"]
    assert "--nproc-per-node=4" in cmd and "--master-addr=127.0.0.1" in cmd and "--master-port=29999" in cmd
    # nothing the launcher's parser could prefix-match (--m, --n) follows the script name; the rest is forwarded
    assert cmd[-2:] == ["--gpus", "4"] and cmd[-3].endswith("bench.py")
    assert json.loads(os.environ.pop("SQB_BENCH_ARGV")) == argv


def test_launcher_parser_accepts_the_spawn_command():
    """torch.distributed.run must parse the command line bench.py builds (its parser rejects `--m` / `--n`
    after the script name as ambiguous prefixes of its own options)."""
    import os
    sys.path.insert(0, str(ROOT))
    import bench
    from torch.distributed.run import get_args_parser
    cmd = bench.spawn_command(2, ["--gpus", "2", "--m", "4096", "--n", "8", "--no-sweep"], port=29998)
    os.environ.pop("SQB_BENCH_ARGV")
    ns = get_args_parser().parse_args(cmd[3:])
    assert ns.training_script.endswith("bench.py") and ns.training_script_args == ["--gpus", "2"]
    # the driver's own launch line parses as well
    ns = get_args_parser().parse_args(["--nnodes=1", "--nproc-per-node", "8", "--master-addr", "127.0.0.1",
                                       "--master-port", "29500", "bench.py", "--gpus", "8", "--steps", "20",
                                       "--warmup", "3"])
    assert ns.training_script_args == ["--gpus", "8", "--steps", "20", "--warmup", "3"]
    ns = get_args_parser().parse_args(["--nnodes=1", "--nproc-per-node", "8", "--master-addr", "127.0.0.1",
                                       "--master-port", "29500", "bench.py", "--impl", "reference", "--gpus", "8",
                                       "--steps", "20", "--warmup", "3"])
    assert ns.training_script_args[:2] == ["--impl", "reference"]
