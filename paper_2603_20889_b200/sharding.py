"""Row-sharded (multi-GPU) orchestration: one process per GPU, rows split into contiguous slabs,
only n x n matrices cross the interconnect.

The reference has no distributed code; this is its k-block structure one level up
(reference src/tsqr.cpp:175-195: k block triangles stacked into Y, one more block QR of Y;
src/gram.cpp:81-92: block partials summed).  Two interchangeable transports exist:

* the C ABI's ``sqb_*_sharded_dev`` entry points (NCCL resolved inside libskinnyqr_b200.so), used by
  ``bench.py``;
* the functions below, which run the same exchange through ``torch.distributed`` (NCCL on GPUs,
  gloo in the CPU tests) around pluggable local kernels.  The local kernels are always supplied by
  the caller - on a GPU box they are the CUDA entry points of ``Context``; nothing here computes.
"""
from __future__ import annotations

from typing import Callable, Tuple


def slab_bounds(m: int, world: int, rank: int) -> Tuple[int, int]:
    """Rows [lo, hi) owned by `rank`: contiguous slabs of ceil(m / world) rows, the last ones short
    or empty (same rule as PanelPlan::block_begin/end, reference include/skinnyqr/plan.hpp:24-37,
    with k = world and b = 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    per = -(-m // world)
    return min(rank * per, m), min((rank + 1) * per, m)


def tsqr_qless_sharded(x_local, local_qr: Callable, stack_qr: Callable, dist, group=None):
    """R of the row-sharded matrix whose slab on this rank is `x_local` (m_local x n).

    local_qr(x_local) -> n x n un-normalised triangle of the slab (zeros for an empty slab);
    stack_qr(y)       -> sign-normalised triangle of the (world*n) x n stack of triangles.
    Every rank returns the same R (all-gather + redundant final combine)."""
    import torch

    r_local = local_qr(x_local)
    world = dist.get_world_size(group)
    n = r_local.shape[0]
    pieces = [torch.empty_like(r_local) for _ in range(world)]
    dist.all_gather(pieces, r_local.contiguous(), group=group)
    y = torch.cat([p.reshape(n, n) for p in pieces], dim=0)  # rank g's triangle at rows [g*n, g*n+n)
    return stack_qr(y)


def gram_sharded(x_local, local_gram: Callable, dist, group=None):
    """Sum over ranks of the slab Gram matrices (all-reduce of n*n doubles)."""
    c = local_gram(x_local).contiguous()
    dist.all_reduce(c, op=dist.ReduceOp.SUM, group=group)
    return c


def cholqr2_sharded(x_local, gram: Callable, gram_solve: Callable, cholesky: Callable,
                    tri_multiply: Callable, dist, group=None):
    """Cholesky-QR2 over row slabs: two streaming passes, two all-reduces, factorisations replicated
    on every rank (reference gram_qr.cpp:123-131)."""
    c1 = gram_sharded(x_local, gram, dist, group)
    r1 = cholesky(c1)
    c2 = gram_sharded(x_local, lambda xl: gram_solve(xl, r1), dist, group)
    r2 = cholesky(c2)
    return tri_multiply(r2, r1)
