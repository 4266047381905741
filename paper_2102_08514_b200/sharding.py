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


def gather_results(local: torch.Tensor, n_total: int, group=None, out: torch.Tensor | None = None) -> torch.Tensor:
    """All-gather the per-rank result shards (shard_range order) into one tensor: one
    all_gather_into_tensor of max-shard-width buffers (NCCL over NVLink); when every shard has
    the same width (n_total divisible by the world size) the gathered buffer IS the result (no
    compaction copy).  `out` (world * width elements) may be passed to reuse a buffer."""
    world = dist.get_world_size(group)
    sizes = [shard_range(n_total, r, world) for r in range(world)]
    width = max(b - a for a, b in sizes)
    if local.shape[0] == width:
        padded = local.contiguous()
    else:
        padded = torch.zeros(width, dtype=local.dtype, device=local.device)
        padded[: local.shape[0]] = local
    full = out if out is not None else torch.empty(world * width, dtype=local.dtype, device=local.device)
    dist.all_gather_into_tensor(full, padded, group=group)
    if all(b - a == width for a, b in sizes):
        return full[:n_total]
    return torch.cat([full[r * width: r * width + (b - a)] for r, (a, b) in enumerate(sizes)])


# ---------------------------------------------------------------------------------------
# Slab partition ("alternative for lattices too big to replicate"): the
# lattice is cut along axis 0 into one slab of unit cells per rank, each rank stores its slab
# plus a halo covering the plan's site reach, query points are routed to the rank owning
# their unit cell with one all-to-all (12 or 24 bytes per point), evaluated there against the
# local slab and routed back with a second all-to-all (4 or 8 bytes per point).


def halo_cells(plan) -> int:
    """Unit cells beyond a slab that a point inside it may read along axis 0: the plan's
    coset-cell reach (plan.site_reach) times the coset spacing, plus one spacing for the
    point's own coset frame."""
    lo, hi = plan.site_reach()
    d = plan.diag[0]
    return (max(abs(lo[0]), abs(hi[0])) + 1) * d


class SlabPartition:
    """Axis-0 slab decomposition of the global grid CoefficientGrid.zeros(cosets, lo, hi)
    (sites with real coordinates in [lo, hi]) over `world` ranks.

    Rank r owns the points whose unit cell floor(x0), clamped into [lo0, hi0], lies in
    [bounds[r], bounds[r+1]); its local grid covers [max(lo0, bounds[r] - halo),
    min(hi0, bounds[r+1] - 1 + halo)] along axis 0 and the full range along the other axes,
    so every site such a point reads is stored locally (interior slab faces) or the read is
    resolved by the boundary policy at a face the slab shares with the global grid.  Exact
    for the 'zero' and 'clamp' policies; 'mirror' reflects indices about the global faces,
    which a slab cannot resolve for points far outside, so it is rejected for world > 1."""

    def __init__(self, cosets, lo, hi, world: int, halo: int, boundary: str = "zero"):
        if world < 1:
            raise ValueError("world must be >= 1")
        if boundary == "mirror" and world > 1:
            raise NotImplementedError("slab partition: the 'mirror' policy needs the replicated lattice")
        self.cosets, self.world, self.halo, self.boundary = cosets, world, int(halo), boundary
        self.lo, self.hi = [int(v) for v in lo], [int(v) for v in hi]
        n0 = self.hi[0] - self.lo[0] + 1
        self.bounds = [self.lo[0] + shard_range(n0, r, world)[0] for r in range(world)] + [self.hi[0] + 1]

    def local_range(self, rank: int) -> tuple:
        """(lo, hi) real-coordinate bounds of rank's local grid."""
        a, b = self.bounds[rank], self.bounds[rank + 1]
        lo = [max(self.lo[0], a - self.halo)] + self.lo[1:]
        hi = [min(self.hi[0], b - 1 + self.halo)] + self.hi[1:]
        return lo, hi

    def owner(self, pts: torch.Tensor) -> torch.Tensor:
        """Owning rank of every point (int64, same device)."""
        c = torch.floor(pts[:, 0].to(torch.float64)).nan_to_num(nan=float(self.lo[0]))
        c = c.clamp(self.lo[0], self.hi[0]).to(torch.int64)
        edges = torch.tensor(self.bounds[1:-1], dtype=torch.int64, device=pts.device)
        return torch.bucketize(c, edges, right=True)

    def local_views(self, grid, rank: int) -> tuple:
        """(arrays, origins) of rank's slab cut out of a global grid's coset arrays (views)."""
        from .runtime import grid_extents

        lo, hi = self.local_range(rank)
        origins, shapes = grid_extents(self.cosets, lo, hi)
        arrays = []
        for k, a in enumerate(grid.arrays):
            o = origins[k][0] - grid.origins[k][0]
            arrays.append(a[o:o + shapes[k][0]])
        return arrays, origins

    def evaluate(self, pts: torch.Tensor, evaluate_local, group=None) -> torch.Tensor:
        """Values at this rank's points `pts` (n, 3), in their order: route each point to its
        owner (all-to-all), evaluate the received points with evaluate_local(points) -> values
        on the local slab, route the values back (all-to-all)."""
        if self.world == 1:
            return torch.as_tensor(evaluate_local(pts), device=pts.device).to(pts.dtype)
        n = pts.shape[0]
        own = self.owner(pts)
        order = torch.argsort(own, stable=True)
        send = pts[order].contiguous()
        counts = torch.bincount(own, minlength=self.world).to(torch.int64)
        recv_counts = torch.empty_like(counts)
        dist.all_to_all_single(recv_counts, counts, group=group)
        sc, rc = counts.tolist(), recv_counts.tolist()
        recv = torch.empty((sum(rc), pts.shape[1]), dtype=pts.dtype, device=pts.device)
        dist.all_to_all_single(recv.view(-1), send.view(-1), output_split_sizes=[c * pts.shape[1] for c in rc],
                               input_split_sizes=[c * pts.shape[1] for c in sc], group=group)
        vals = evaluate_local(recv)
        vals = torch.as_tensor(vals, device=pts.device).to(pts.dtype).contiguous()
        back = torch.empty(n, dtype=vals.dtype, device=pts.device)
        dist.all_to_all_single(back, vals, output_split_sizes=sc, input_split_sizes=rc, group=group)
        out = torch.empty_like(back)
        out[order] = back
        return out
