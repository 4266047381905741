"""Per-step e2e timings of the pinned-host pipeline + a CUDA trace of a few steps."""
import json
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    _, grid, pts, interp = bench.make_workload("tricubic_cc256_fp32", 0, dev)
    n = pts.shape[0]
    hp = pts.cpu().pin_memory()
    ho = torch.empty(n, dtype=grid.dtype).pin_memory()

    def step():
        interp.eval_batch(grid, hp, out=ho, check=False, order="morton")

    times = []
    for _ in range(12):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        step()
        e.record()
        torch.cuda.synchronize()
        times.append(round(s.elapsed_time(e), 1))
    print("step ms:", times, flush=True)
    from torch.profiler import ProfilerActivity, profile

    with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
        for _ in range(4):
            step()
        torch.cuda.synchronize()
    prof.export_chrome_trace("gpurun_out/e2e_trace.json")
    print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=15))


if __name__ == "__main__":
    main()
