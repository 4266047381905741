"""Kernel breakdown of the public device-tensor call eval_batch(grid, pts, order='morton')
(torch.profiler / CUPTI) next to its CUDA-event time.

    python tools/public_call_timing.py [--workload W]
"""
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
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    plan, grid, pts, interp = bench.make_workload(a.workload, 0, dev)
    out = torch.empty(pts.shape[0], dtype=grid.dtype, device=dev)

    def call():
        interp.eval_batch(grid, pts, out=out, check=False, order="morton")

    for _ in range(3):
        call()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        call()
    e1.record()
    torch.cuda.synchronize()
    print(f"{a.workload}: public morton call {e0.elapsed_time(e1) / 10:.3f} ms")
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA, torch.profiler.ProfilerActivity.CPU]) as prof:
        call()
        torch.cuda.synchronize()
    print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=15))


if __name__ == "__main__":
    main()
