"""Multi-GPU sharding of the reconstruction.

Query points are independent, so each rank evaluates a contiguous shard of the points
against its own replica of the lattice (67–535 MB, tiny next to 180 GB of HBM).  There
is no collective on the data path; `gather_results` (an all-gather of n·sizeof(T)
bytes over NCCL/NVLink) runs only when the caller asks for one output tensor.
"""

from __future__ import annotations

import torch
import torch.distributed as dist


def shard_range(n: int, rank: int, world: int) -> tuple:
    """[start, end) of rank's contiguous shard; shards differ in size by at most one."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, extra = divmod(n, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def shard_points(pts: torch.Tensor, rank: int, world: int) -> torch.Tensor:
    a, b = shard_range(pts.shape[0], rank, world)
    return pts[a:b]


def gather_results(local: torch.Tensor, n_total: int, group=None) -> torch.Tensor:
    """All-gather the per-rank result shards (shard_range order) into one tensor."""
    world = dist.get_world_size(group)
    sizes = [shard_range(n_total, r, world) for r in range(world)]
    width = max(b - a for a, b in sizes)
    padded = torch.zeros(width, dtype=local.dtype, device=local.device)
    padded[: local.shape[0]] = local
    parts = [torch.empty_like(padded) for _ in range(world)]
    dist.all_gather(parts, padded, group=group)
    return torch.cat([p[: b - a] for p, (a, b) in zip(parts, sizes)])
