"""One protocol-B evaluation (order='sort') of a bench workload with iid points, for a
kernel launch list under ncu:  python tools/protocol_b_once.py --workload tricubic_cc256_fp32"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default=bench.HEADLINE)
    ap.add_argument("--gather", type=int, default=0)
    ap.add_argument("--unordered", type=int, default=0)
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    plan, grid, pts, interp = bench.make_workload(a.workload, 0, dev, order="random")
    interp.sort_gather = bool(a.gather)
    out = torch.empty(pts.shape[0], dtype=grid.dtype, device=dev)
    def step():
        if a.unordered:
            interp.eval_batch_unordered(grid, pts, check=False)
        else:
            interp.eval_batch(grid, pts, out=out, check=False, order="sort")

    step()
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStart()
    step()
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStop()


if __name__ == "__main__":
    main()
