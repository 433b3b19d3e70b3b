"""Host-side wiring of the row-sharded (multi-GPU) runs: one process per GPU, rows split into
contiguous slabs, only n x n matrices cross the interconnect.

The reference has no distributed code; the protocol is its k-block structure one level up
(reference src/tsqr.cpp:175-195: k block triangles stacked into Y, one more block QR of Y;
src/gram.cpp:81-92: block partials summed in ascending order) and it is implemented ONCE, in the
C library (``sqb_*_sharded_dev``: local pass -> all-gather of n x n blocks -> combine kernels).
This module only provides what a launcher needs around it - nothing here computes:

* ``slab_bounds``      which rows a rank owns;
* ``attach``           gives a ``Context`` its transport: NCCL inside the library (communicator
                       id broadcast through ``torch.distributed``) when the process group runs on
                       NCCL, otherwise ``TorchExchange``;
* ``TorchExchange``    the library's all-gather hook (``sqb_set_allgather``) served by any
                       ``torch.distributed`` backend through host staging - this is how the C
                       drivers are exercised with world > 1 on one GPU (gloo) and how an MPI-style
                       host transport would plug in;
* ``max_over_ranks``   the bench's timing reduction.

``bench.py`` and the multi-rank tests use exactly these functions.
"""
from __future__ import annotations

from typing import Tuple

import numpy as np


def slab_bounds(m: int, world: int, rank: int) -> Tuple[int, int]:
    """Rows [lo, hi) owned by `rank`: contiguous slabs of ceil(m / world) rows, the last ones short
    or empty (same rule as PanelPlan::block_begin/end, reference include/skinnyqr/plan.hpp:24-37,
    with k = world and b = 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    per = -(-m // world)
    return min(rank * per, m), min((rank + 1) * per, m)


def _backend_device(dist, group=None):
    """Tensors handed to the collectives of this process group live on this device."""
    import torch
    if dist.get_backend(group) == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def broadcast_bytes(payload, dist, src=0, group=None) -> bytes:
    """`payload` (bytes on rank `src`, ignored elsewhere) -> the same bytes on every rank."""
    box = [payload if dist.get_rank(group) == src else None]
    dist.broadcast_object_list(box, src=src, group=group)
    return bytes(box[0])


def max_over_ranks(value: float, dist, group=None) -> float:
    """Slowest rank's figure (bench contract: device time, max over ranks)."""
    import torch
    if dist is None or not dist.is_initialized() or dist.get_world_size(group) == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=_backend_device(dist, group))
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


class TorchExchange:
    """All-gather of `count` doubles per rank through torch.distributed.

    ``gather_host`` is the transport proper (host arrays in, host array out); ``__call__`` is the
    signature the library's hook expects (device addresses): it stages through host memory with
    the context's stream-ordered copies, so the gathered blocks are valid for everything the
    library enqueues afterwards."""

    def __init__(self, dist, group=None, ctx=None):
        self.dist, self.group, self.ctx = dist, group, ctx
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.calls = 0

    def gather_host(self, block: np.ndarray) -> np.ndarray:
        """(count,) float64 on every rank -> (world, count): row g is rank g's block."""
        import torch
        dev = _backend_device(self.dist, self.group)
        send = torch.from_numpy(np.ascontiguousarray(block, dtype=np.float64)).to(dev)
        pieces = [torch.empty_like(send) for _ in range(self.world)]
        self.dist.all_gather(pieces, send, group=self.group)
        self.calls += 1
        return torch.stack(pieces).cpu().numpy()

    def __call__(self, send_ptr: int, recv_ptr: int, count: int) -> int:
        send = np.empty(count, dtype=np.float64)
        self.ctx.copy_d2h(send, send_ptr)
        gathered = np.ascontiguousarray(self.gather_host(send))
        self.ctx.copy_h2d(recv_ptr, gathered)
        return 0


def attach(ctx, dist, group=None, transport: str = "auto"):
    """Make `ctx` a member of the process group: afterwards ``ctx.*_sharded`` run over all ranks.

    transport "nccl": the library's own NCCL communicator (rank 0 creates the unique id, it is
    broadcast through the process group); "torch": ``TorchExchange`` over whatever backend the
    group uses; "auto": NCCL when the group itself runs on NCCL.  Returns the transport's name."""
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    if transport == "auto":
        transport = "nccl" if dist.get_backend(group) == "nccl" else "torch"
    if transport == "nccl":
        uid = broadcast_bytes(ctx.nccl_unique_id() if rank == 0 else None, dist, 0, group)
        ctx.init_nccl(uid, rank, world)
    elif transport == "torch":
        ctx.exchange = TorchExchange(dist, group, ctx)
        ctx.set_allgather(ctx.exchange, rank, world)
    else:
        raise ValueError(f"unknown transport {transport!r}")
    return transport
