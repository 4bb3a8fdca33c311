"""Multi-GPU plumbing for the MASQuant hot path: one process per GPU,
torch.distributed for the exchanges.  The path shards naturally:

  * calibration (A1) and the loss (A8) by token rows: each rank processes its own tokens;
    the only exchanges are an all-reduce MAX of the per-modality ranges R (max is
    order-free, so R is bit-identical to one process) and SUMs of the token counts and of the
    per-modality loss sums, after which masq_loss_finalize forms the loss;
  * the forward (A4-A7) by output columns through pointer offsets (column_shards).

No data-path collective is needed anywhere else, and the messages are tens of KB, so NCCL's
all-reduce is used as is (no fused compute+collective kernel is warranted).
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def world():
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(), dist.get_world_size()
    return 0, 1


def token_shard(T: int, rank: int, world_size: int, align: int = 1024):
    """Contiguous token block of this rank, aligned to `align` tokens (whole samples)."""
    units = -(-T // align)
    per = -(-units // world_size)
    a = min(T, rank * per * align)
    b = min(T, (rank + 1) * per * align)
    return a, b


def column_shards(n: int, world_size: int, align: int = 32):
    """[(j0, j1)] output-column ranges (multiples of `align`) covering n for world_size ranks."""
    units = n // align
    per, extra = divmod(units, world_size)
    out, j = [], 0
    for r in range(world_size):
        w = (per + (1 if r < extra else 0)) * align
        out.append((j, j + w))
        j += w
    return out


def reduce_stats(R_list, counts, group=None):
    """All-reduce every linear's R (MAX) and the token counts (SUM), in two batched calls.

    R_list: list of float32 [M x d] tensors that are views of ONE flat buffer is the fast path
    (pass that buffer as a single-element list); counts: int64 tensor."""
    _, ws = world()
    if ws == 1:
        return
    for R in R_list:
        dist.all_reduce(R, op=dist.ReduceOp.MAX, group=group)
    dist.all_reduce(counts, op=dist.ReduceOp.SUM, group=group)


def reduce_loss(sums, counts, group=None):
    """All-reduce the per-modality loss sums (f64) and counts (i64): SUM."""
    _, ws = world()
    if ws == 1:
        return
    dist.all_reduce(sums, op=dist.ReduceOp.SUM, group=group)
    dist.all_reduce(counts, op=dist.ReduceOp.SUM, group=group)


def reduce_grad(grad, group=None):
    """All-reduce the N1 gradient (f64 [M x d]): SUM.  Each rank's grad must have been formed
    with the GLOBAL token counts (masq_calib_loss_grad's count_norm), so the sum is the
    gradient of the whole batch's loss."""
    _, ws = world()
    if ws == 1:
        return
    dist.all_reduce(grad, op=dist.ReduceOp.SUM, group=group)


def reduce_gram(G, group=None):
    """All-reduce the CMC Gram matrices (f64 [M-1 x d x d], N2): SUM over the token shards."""
    _, ws = world()
    if ws == 1:
        return
    dist.all_reduce(G, op=dist.ReduceOp.SUM, group=group)


def max_over_ranks(x: float, device=None) -> float:
    """Max of a host float over ranks (timings: the slowest rank defines the step)."""
    _, ws = world()
    if ws == 1:
        return x
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
