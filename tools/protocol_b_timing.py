"""Protocol B stage timings (CUDA events): the whole eval_batch(order='sort') call and, on the
same inputs, the payload sort and the brick evaluation alone.

    python tools/protocol_b_timing.py [--workload W] [--iters 10]
"""
import argparse
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2102_08514_b200 import _native  # noqa: E402
from paper_2102_08514_b200.runtime import _sort_frame  # noqa: E402


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
    plan, grid, pts, interp = bench.make_workload(a.workload, 0, dev)  # Morton order
    shuffled = pts[torch.randperm(pts.shape[0], device=dev)]
    n = pts.shape[0]
    out = torch.empty(n, dtype=grid.dtype, device=dev)
    lib = _native.lib()
    dtype = _native.SP_F32 if grid.dtype == torch.float32 else _native.SP_F64
    b = interp.brick_log2(grid)
    (lo0, lo1, lo2), bits = _sort_frame(grid, b)
    t_call = timed(lambda: interp.eval_batch(grid, shuffled, out=out, check=False, order="sort"), a.iters)
    sp_ = torch.empty_like(pts)
    perm = torch.empty(n, dtype=torch.int32, device=dev)
    start = torch.empty(n + 1, dtype=torch.int64, device=dev)
    count = torch.empty(1, dtype=torch.int32, device=dev)
    tmp = torch.empty(int(lib.sp_sort_points_payload_temp_bytes(n, dtype)), dtype=torch.uint8, device=dev)
    st = torch.cuda.current_stream(dev).cuda_stream

    def sort():
        _native.check(lib.sp_sort_points_payload(shuffled.data_ptr(), n, dtype, lo0, lo1, lo2, bits, b, sp_.data_ptr(),
                                                 perm.data_ptr(), start.data_ptr(), count.data_ptr(), tmp.data_ptr(),
                                                 tmp.numel(), st))

    t_sort = timed(sort, a.iters)
    import time

    torch.cuda.synchronize()
    t0 = time.perf_counter()
    sort()
    t_host = (time.perf_counter() - t0) * 1e3
    torch.cuda.synchronize()
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
        sort()
        torch.cuda.synchronize()
    print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=12))
    print(f"payload sort: host enqueue {t_host:.3f} ms")
    h = interp._handle(dev)
    gdesc = grid.descriptor()

    def ev(scatter):
        if scatter:
            _native.check(lib.sp_eval_bricks_perm32(h, ctypes.byref(gdesc), sp_.data_ptr(), n, dtype, start.data_ptr(),
                                                    count.data_ptr(), n, b, perm.data_ptr(), out.data_ptr(), None, st))
        else:
            _native.check(lib.sp_eval_bricks_dev(h, ctypes.byref(gdesc), sp_.data_ptr(), n, dtype, start.data_ptr(),
                                                 count.data_ptr(), n, b, None, out.data_ptr(), None, st))

    t_eval_scatter = timed(lambda: ev(True), a.iters)
    t_eval = timed(lambda: ev(False), a.iters)
    t_morton = timed(lambda: interp.eval_batch(grid, interp.prepare(grid, pts, presorted=True), out=out, check=False),
                     a.iters)
    print(f"{a.workload}: n={n} call(order=sort) {t_call:.3f} ms = {n / t_call / 1e6:.2f} Gpts/s | payload sort "
          f"{t_sort:.3f} | eval brick-sorted + scatter {t_eval_scatter:.3f} | eval no scatter {t_eval:.3f} | "
          f"Morton-ordered (protocol A) {t_morton:.3f}")


if __name__ == "__main__":
    main()
