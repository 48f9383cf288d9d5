"""Multi-GPU partitioning of the conv path along its natural shards.

The path has no exchange step: a large single op is split by batch (each rank convolves
a contiguous N/g slice with the full, replicated weights), and a sweep of independent
ops is split by longest-processing-time-first assignment on predicted roofline time.
The only communication is control: a barrier around the timed region, a max-over-ranks
of the measured time, and a gather of results to rank 0 after timing.  One process per
GPU; torch.distributed (NCCL on GPUs, gloo in the CPU tests) carries these.
"""

from __future__ import annotations

import heapq
from dataclasses import replace
from typing import Callable, Sequence


def batch_shard(n_total: int, world: int, rank: int) -> tuple[int, int]:
    """(first image, image count) of `rank`'s contiguous slice; sizes differ by <= 1."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of {world}")
    base, extra = divmod(n_total, world)
    start = rank * base + min(rank, extra)
    return start, base + (1 if rank < extra else 0)


def shard_descriptor(desc, world: int, rank: int):
    """The descriptor of `rank`'s batch slice (None if the slice is empty)."""
    _, count = batch_shard(desc.batch, world, rank)
    return replace(desc, batch=count) if count else None


def lpt_assign(costs: Sequence[float], world: int) -> list[list[int]]:
    """Longest-processing-time-first: ops sorted by decreasing cost go to the least
    loaded rank (ties -> lowest rank; equal costs keep index order).  Deterministic, so
    every rank computes the same partition without communicating."""
    order = sorted(range(len(costs)), key=lambda i: (-costs[i], i))
    heap = [(0.0, r) for r in range(world)]
    out: list[list[int]] = [[] for _ in range(world)]
    for i in order:
        load, r = heapq.heappop(heap)
        out[r].append(i)
        heapq.heappush(heap, (load + costs[i], r))
    return [sorted(x) for x in out]


def sweep_partition(descs: Sequence, world: int, cost: Callable[[object], float]) -> list[list[int]]:
    return lpt_assign([cost(d) for d in descs], world)


def max_over_ranks(value: float, dist=None) -> float:
    """Max of a per-rank scalar (the timed region's duration) over all ranks."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return value
    import torch
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([float(value)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(value: float, dist=None) -> float:
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return value
    import torch
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([float(value)], dtype=torch.float64, device=dev)
    dist.all_reduce(t)
    return float(t.item())


def gather_to_rank0(obj, dist=None):
    """Python-object gather after the timed region (results, CSV rows)."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return [obj]
    out = [None] * dist.get_world_size()
    dist.all_gather_object(out, obj)
    return out if dist.get_rank() == 0 else None
