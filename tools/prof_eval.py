"""Profiling driver: run one workload's eval_batch a few times (for ncu / sanitizer).

    python tools/prof_eval.py --workload tricubic_cc256_fp32 [--points N] [--iters 3] [--order morton|random]
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
    ap.add_argument("--points", type=int, default=None)
    ap.add_argument("--iters", type=int, default=3)
    ap.add_argument("--order", default="morton")
    ap.add_argument("--mode", default="brick", choices=["brick", "chunk"])
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    plan, grid, pts, interp = bench.make_workload(a.workload, 0, dev, order=a.order, n_override=a.points)
    out = torch.empty(pts.shape[0], dtype=grid.dtype, device=dev)
    if a.mode == "brick":
        pts = interp.prepare(grid, pts, presorted=(a.order == "morton"))
    for _ in range(a.iters):
        interp.eval_batch(grid, pts, out=out, check=False)
    torch.cuda.synchronize()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    start.record()
    for _ in range(a.iters):
        interp.eval_batch(grid, pts, out=out, check=False)
    end.record()
    torch.cuda.synchronize()
    ms = start.elapsed_time(end) / a.iters
    import ctypes

    from paper_2102_08514_b200 import _native

    lib = _native.lib()
    buf = (ctypes.c_uint64 * 4)()
    lib.sp_debug_stats(1, None)
    interp.eval_batch(grid, pts, out=out, check=False)
    torch.cuda.synchronize()
    lib.sp_debug_stats(0, buf)
    st, un, el = buf[0], buf[1], buf[2]
    n = out.shape[0]
    print(f"{a.workload} [{a.mode}] kernel={interp.kernel_name()} n={n} {ms:.3f} ms  "
          f"{n / ms / 1e6:.2f} Gpts/s  staged={st} unstaged={un} "
          f"elems/pt={el / max(1, n):.2f} env=({os.environ.get('SP_PPT', '-')},{os.environ.get('SP_TILE_KB', '-')})")


if __name__ == "__main__":
    main()
