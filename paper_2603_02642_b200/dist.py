"""Multi-GPU plumbing for the instance-sharded inner solve.

Instances are independent: rank r of N owns a contiguous range
of instances and its own nrto handle; no data-path collective exists.  The
only collectives are the max-over-ranks step time and the batch-wide
residual statistics (max r_p, #unconverged, any diverged), done through
torch.distributed (NCCL over NVLink on the GPU box, gloo in CPU tests).
"""
from __future__ import annotations


def instance_range(rank: int, world: int, per_rank: int):
    """(first instance, count) of rank `rank` under weak scaling."""
    if not (0 <= rank < world) or per_rank < 1:
        raise ValueError("bad rank/world/per_rank")
    return rank * per_rank, per_rank


def strong_range(rank: int, world: int, total: int):
    """(first, count) of a contiguous split of `total` instances (strong scaling)."""
    base, rem = divmod(total, world)
    first = rank * base + min(rank, rem)
    return first, base + (1 if rank < rem else 0)


def max_over_ranks(value: float, device=None) -> float:
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def batch_stats(r_p, status, device=None):
    """Batch-wide residual reduction: (max r_p, #unconverged, any diverged)."""
    import torch
    import torch.distributed as dist
    r_p = torch.as_tensor(r_p, device=device)
    status = torch.as_tensor(status, device=device)
    mx = torch.tensor([r_p.max().item() if r_p.numel() else 0.0], dtype=torch.float64,
                      device=device)
    cnt = torch.tensor([float((status != 0).sum().item()), float((status == 2).any().item())],
                       dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        dist.all_reduce(cnt, op=dist.ReduceOp.SUM)
    return float(mx.item()), int(cnt[0].item()), bool(cnt[1].item() > 0)
