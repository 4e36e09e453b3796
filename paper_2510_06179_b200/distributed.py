"""K5 host side: batch sharding across GPUs and the theta-gradient exchange.

OCP instances are independent, so each rank owns a fixed
contiguous range of instances — the reference's parallel_for chunking
(common.hpp:84-97) lifted to ranks — and keeps its warm-start caches
rank-local across epochs. The only cross-GPU traffic per training step is the
summed learnable theta-gradient plus the loss scalar (train.hpp:126-131):
each rank sums its shard in instance order on the device (il_sum_kernel), the
partial sums are all-gathered over NCCL (NVLink/NVSwitch) and every rank adds
them in rank order, so all ranks hold bit-identical sums.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard_range(n: int, rank: int, world: int):
    """[lo, hi) of rank's instances: ceil-sized contiguous chunks."""
    chunk = (n + world - 1) // world
    lo = min(n, rank * chunk)
    return lo, min(n, lo + chunk)


def global_batch(batch: int, world: int, scaling: str) -> int:
    """Problems in the whole job: `batch` per rank (weak scaling) or `batch`
    split over the ranks (strong scaling)."""
    if scaling not in ("weak", "strong"):
        raise ValueError(f"scaling must be weak or strong, not {scaling!r}")
    return batch * world if scaling == "weak" else batch


def max_over_ranks(x: float, device=None, group=None) -> float:
    """The largest `x` over all ranks (a step time: the job ends with its
    slowest rank)."""
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size(group) == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def fixed_order_allreduce(partial: torch.Tensor, group=None) -> torch.Tensor:
    """Sum of every rank's `partial`, added in rank order on every rank
    (0.0 + p_0 + p_1 + ...): deterministic and identical across ranks."""
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size(group) == 1:
        return partial.clone()
    world = dist.get_world_size(group)
    bufs = [torch.empty_like(partial) for _ in range(world)]
    dist.all_gather(bufs, partial.contiguous(), group=group)
    out = torch.zeros_like(partial)
    for b in bufs:
        out = out + b
    return out
