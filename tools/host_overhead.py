"""Host-side cost of one PlanInterpreter.eval_batch call (tiny batches, so the GPU is idle
and the wall clock is the Python + ctypes + launch path).  python tools/host_overhead.py"""
import sys
import time

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    for name in ("trilinear_cc64_fp32", "tricubic_cc256_fp32", "fcc6_4x161_fp32"):
        _, grid, pts, interp = bench.make_workload(name, 0, dev, n_override=4096)
        batch = interp.prepare(grid, pts, presorted=True)
        out = torch.empty(pts.shape[0], dtype=grid.dtype, device=dev)
        for _ in range(20):
            interp.eval_batch(grid, batch, out=out, check=False)
        torch.cuda.synchronize()
        t = time.perf_counter()
        n = 2000
        for _ in range(n):
            interp.eval_batch(grid, batch, out=out, check=False)
        torch.cuda.synchronize()
        print(f"{name}: {(time.perf_counter() - t) / n * 1e6:.1f} us per eval_batch(PointBatch) call")
        _, grid, pts, interp = bench.make_workload(name, 0, dev, n_override=1_000_000)
        batch = interp.prepare(grid, pts, presorted=True)
        out = torch.empty(pts.shape[0], dtype=grid.dtype, device=dev)
        ms = bench.measure(lambda: interp.eval_batch(grid, batch, out=out, check=False), 200, 5,
                           torch.cuda.current_stream(dev))
        print(f"   1e6 points: {ms * 1e3:.1f} us/step -> {1e6 / ms / 1e6:.1f} Gpts/s")


if __name__ == "__main__":
    main()
