"""Protocol-B timing for one SP_SORT_BEGIN_BIT setting (set in the environment; the library
reads it once): order='sort' and eval_batch_unordered on iid points of a bench workload,
with a bit-identity check against the chunk kernel.
    SP_SORT_BEGIN_BIT=3 python tools/sort_bits_probe.py [--workload W] [--iters 10]"""
import argparse
import json
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
    ap.add_argument("--iters", type=int, default=10)
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    plan, grid, pts, interp = bench.make_workload(a.workload, 0, dev, order="random")
    out = torch.empty(pts.shape[0], dtype=grid.dtype, device=dev)
    ms_sort = timed(lambda: interp.eval_batch(grid, pts, out=out, check=False, order="sort"), a.iters)
    ms_unord = timed(lambda: interp.eval_batch_unordered(grid, pts, check=False), a.iters)
    m = 1 << 22
    want = interp.eval_batch(grid, pts[:m], order="given")
    got = interp.eval_batch(grid, pts[:m], order="sort")
    vals, perm = interp.eval_batch_unordered(grid, pts[:m])
    print(json.dumps({"workload": a.workload, "begin_bit": os.environ.get("SP_SORT_BEGIN_BIT", "0"),
                      "sort_ms": round(ms_sort, 3), "unordered_ms": round(ms_unord, 3),
                      "bit_identical": bool(torch.equal(got, want) and torch.equal(vals, want[perm]))}), flush=True)


if __name__ == "__main__":
    main()
