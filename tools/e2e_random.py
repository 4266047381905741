"""End-to-end throughput from pinned HOST points in random (generation) order through the
default eval_batch (order="auto" -> per-chunk GPU sort in the pinned-host pipeline), next to
the Morton-ordered input of bench.py's e2e line.  python tools/e2e_random.py [workload]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else bench.HEADLINE
    dev = torch.device("cuda", 0)
    for order in ("random", "morton"):
        plan, grid, pts, interp = bench.make_workload(name, 0, dev, order=order)
        host = pts.cpu().pin_memory()
        out = torch.empty(pts.shape[0], dtype=grid.dtype).pin_memory()
        del pts
        for _ in range(2):
            interp.eval_batch(grid, host, out=out)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            interp.eval_batch(grid, host, out=out)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        print(f"{name} host {order} order: {ms:.2f} ms  {host.shape[0] / ms / 1e6:.2f} Gpts/s", flush=True)


if __name__ == "__main__":
    main()
