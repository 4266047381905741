"""Protocol B call time with each result-scatter variant (CUDA events), and bit-identity.

    python tools/scatter_timing.py [--workload W] [--iters 10]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402


def timed(fn, iters):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / iters


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default=bench.HEADLINE)
    ap.add_argument("--iters", type=int, default=10)
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    plan, grid, pts, interp = bench.make_workload(a.workload, 0, dev)
    shuffled = pts[torch.randperm(pts.shape[0], device=dev)]
    n = pts.shape[0]
    outs = {}
    for name, sorted_scatter in (("sorted-window scatter", True), ("L2-window passes", False)):
        interp.scatter_sorted = sorted_scatter
        out = torch.empty(n, dtype=grid.dtype, device=dev)
        t = timed(lambda: interp.eval_batch(grid, shuffled, out=out, check=False, order="sort"), a.iters)
        outs[name] = out
        print(f"{a.workload}: order=sort with {name}: {t:.3f} ms ({n / t / 1e6:.2f} Gpts/s)")
    v = list(outs.values())
    print("identical:", torch.equal(v[0], v[1]))


if __name__ == "__main__":
    main()
