"""CPU, world_size 2 (gloo): the multi-GPU host logic — sharding and the optional gather."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2102_08514_b200.sharding import gather_results, shard_range


def test_shard_range_partitions():
    for n in (0, 1, 7, 100, 10**8 + 3):
        for world in (1, 2, 3, 8):
            spans = [shard_range(n, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    a, b = shard_range(n, rank, world)
    # stand-in for the per-rank reconstruction: f(i) = 2 i + 1 on the rank's shard
    local = (2 * torch.arange(a, b, dtype=torch.float64) + 1)
    full = gather_results(local, n)
    ok = torch.equal(full, 2 * torch.arange(n, dtype=torch.float64) + 1)
    # max-over-ranks timing reduction used by bench.py
    t = torch.tensor([float(rank + 1)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    q.put((rank, bool(ok), float(t.item())))
    dist.destroy_process_group()


@pytest.mark.parametrize("n", [1001, 8])
def test_gather_and_max_over_ranks_world2(n):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert sorted(r[0] for r in res) == [0, 1]
    assert all(r[1] for r in res)
    assert all(r[2] == 2.0 for r in res)


def _slab_worker(rank, world, port, name, boundary, q):
    """Each rank: its own random points, the slab partition routes them to the ranks owning
    their cells, the owner evaluates on its slab (+ halo) with the oracle, values come back."""
    import numpy as np

    from oracle.plan_numpy import NumpyGrid, PlanTables, eval_batch as oracle_eval
    from paper_2102_08514_b200 import corpus
    from paper_2102_08514_b200.runtime import CoefficientGrid
    from paper_2102_08514_b200.sharding import SlabPartition, halo_cells

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        plan = corpus.build_plan(name)
        _, cos = corpus.lattice_of(name)
        lo, hi = [0, -3, 2], [41, 9, 13]
        grid = CoefficientGrid.zeros(cos, lo, hi, boundary=boundary, device="cpu", dtype=torch.float64)
        rng = np.random.default_rng(99)  # same global data on every rank
        for a in grid.arrays:
            a.copy_(torch.from_numpy(rng.random(tuple(a.shape))))
        part = SlabPartition(cos, lo, hi, world, halo_cells(plan), boundary)
        arrays, origins = part.local_views(grid, rank)
        tables = PlanTables(plan)
        local = NumpyGrid(plan.diag, plan.shifts, [a.numpy() for a in arrays], origins, boundary)

        def evaluate_local(p):
            return torch.from_numpy(oracle_eval(plan, local, p.numpy(), tables))

        prng = np.random.default_rng(1000 + rank)
        pts = np.stack([prng.uniform(-4, 46, 700), prng.uniform(-5, 11, 700), prng.uniform(1, 15, 700)], 1)
        got = part.evaluate(torch.from_numpy(pts), evaluate_local).numpy()
        ng = NumpyGrid(plan.diag, plan.shifts, [a.numpy() for a in grid.arrays], grid.origins, boundary)
        want = oracle_eval(plan, ng, pts, tables)
        # the oracle's monomial sums are BLAS dot products: batch composition changes their
        # rounding (~1e-16), so the slab result is compared to the replicated one at 1e-13
        q.put((rank, bool(np.abs(got - want).max() <= 1e-13 * max(1.0, np.abs(want).max())), float(np.abs(got - want).max())))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,name,boundary", [(2, "bcc_quintic_rd", "zero"), (3, "fcc_cubic", "clamp"),
                                                 (2, "cc_tricubic", "clamp")])
def test_slab_partition_matches_replicated(world, name, boundary):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_slab_worker, args=(r, world, port, name, boundary, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert sorted(r[0] for r in res) == list(range(world))
    assert all(r[1] for r in res), res


def test_slab_partition_geometry():
    from paper_2102_08514_b200 import corpus
    from paper_2102_08514_b200.sharding import SlabPartition, halo_cells

    plan = corpus.build_plan("bcc_quintic_rd")
    _, cos = corpus.lattice_of("bcc_quintic_rd")
    h = halo_cells(plan)
    part = SlabPartition(cos, [0, 0, 0], [99, 9, 9], 4, h)
    assert part.bounds == [0, 25, 50, 75, 100]
    assert part.local_range(0) == ([0, 0, 0], [24 + h, 9, 9]) and part.local_range(3) == ([75 - h, 0, 0], [99, 9, 9])
    own = part.owner(torch.tensor([[-7.0, 0, 0], [24.99, 0, 0], [25.0, 0, 0], [1e9, 0, 0], [float("nan"), 0, 0]]))
    assert own.tolist() == [0, 0, 1, 3, 0]
    with pytest.raises(NotImplementedError):
        SlabPartition(cos, [0, 0, 0], [99, 9, 9], 2, h, "mirror")
