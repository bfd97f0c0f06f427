"""Sample-sharded data parallelism for the hypergradient.

Each rank owns a contiguous block of training samples (their recycle spaces,
bases and solves stay on that rank's GPU).  The only exchange per upper step
is the p-vector hypergradient: every rank all-gathers the per-sample vectors
and sums them in global sample order, so the result is bitwise identical for
1/2/4/8 ranks and equal to the single-process sum.  (An all-reduce would be
cheaper by ~p*B*8 bytes but its summation order depends on the world size.)
The Armijo line search needs one scalar per trial: ``allreduce_cost``.
"""

from __future__ import annotations

import torch
import torch.distributed as dist

__all__ = ["shard", "ordered_sum", "allgather_sum", "allreduce_cost"]


def shard(batch: int, world: int, rank: int) -> range:
    """Contiguous block of samples owned by ``rank`` (sizes differ by at most one)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} for world {world}")
    lo = batch * rank // world
    hi = batch * (rank + 1) // world
    return range(lo, hi)


def ordered_sum(per_sample: torch.Tensor) -> torch.Tensor:
    """Sum of the rows in sample order (the reference's left-to-right accumulation):
    one ``kr_ordered_sum`` launch on CUDA tensors (a thread per entry adding the rows
    left to right), the same row-by-row accumulation elsewhere."""
    if per_sample.is_cuda and per_sample.dtype == torch.float64 and per_sample.dim() == 2:
        from . import _lib

        rows = per_sample.contiguous()
        out = torch.empty(rows.shape[1], dtype=torch.float64, device=rows.device)
        _lib.check(_lib.lib().kr_ordered_sum(rows.data_ptr(), rows.shape[0], rows.shape[1], rows.shape[1],
                                             out.data_ptr(), _lib.stream_ptr()), "kr_ordered_sum")
        _lib.note_launch("kr_ordered_sum")
        return out
    acc = per_sample[0].clone()
    for k in range(1, per_sample.shape[0]):
        acc += per_sample[k]
    return acc


def allgather_sum(local: torch.Tensor, batch: int, group=None) -> torch.Tensor:
    """All-gather the local per-sample hypergradients [b_local, p] and return the
    sample-ordered global sum (identical on every rank)."""
    if not dist.is_available() or not dist.is_initialized():
        return ordered_sum(local)
    world = dist.get_world_size(group)
    p = local.shape[1]
    sizes = [len(shard(batch, world, r)) for r in range(world)]
    cap = max(sizes)
    buf = torch.zeros(cap, p, dtype=local.dtype, device=local.device)
    buf[: local.shape[0]] = local
    out = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(out, buf, group=group)
    rows = torch.cat([o[:s] for o, s in zip(out, sizes)], dim=0)
    return ordered_sum(rows)


def allreduce_cost(value: float, device, group=None) -> float:
    """Sum of per-rank upper costs (one 8-byte all-reduce per Armijo trial)."""
    if not dist.is_available() or not dist.is_initialized():
        return float(value)
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, group=group)
    return float(t.item())
