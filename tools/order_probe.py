"""Throughput of eval_batch by input order on one bench workload: iid points in generation
order through the chunk kernel (order='given'), through the GPU Morton sort (order='sort',
protocol B), and pre-sorted (protocol A, brick kernel only).

    python tools/order_probe.py --workload tricubic_cc256_fp32 [--points N] [--iters 10]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402


def timed(fn, iters):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default=bench.HEADLINE)
    ap.add_argument("--points", type=int, default=None)
    ap.add_argument("--iters", type=int, default=10)
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    plan, grid, pts, interp = bench.make_workload(a.workload, 0, dev, order="random", n_override=a.points)
    n = pts.shape[0]
    out = torch.empty(n, dtype=grid.dtype, device=dev)
    res = {}
    res["given"] = timed(lambda: interp.eval_batch(grid, pts, out=out, check=False, order="given"), a.iters)
    for gather in (False, True):
        interp.sort_gather = gather
        res[f"sort gather={int(gather)}"] = timed(
            lambda: interp.eval_batch(grid, pts, out=out, check=False, order="sort"), a.iters)
    interp.sort_gather = False
    batch = interp.prepare(grid, pts)
    sorted_pts = batch.pts
    pre = interp.prepare(grid, sorted_pts, presorted=True)
    res["morton (A)"] = timed(lambda: interp.eval_batch(grid, pre, out=out, check=False), a.iters)
    for k, ms in res.items():
        print(f"{a.workload} order={k}: {ms:.3f} ms  {n / ms / 1e6:.2f} Gpts/s", flush=True)


if __name__ == "__main__":
    main()
