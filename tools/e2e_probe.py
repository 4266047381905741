"""Probe the host<->device path of the e2e bench line: raw PCIe copy rates (each direction,
and both at once) and PlanInterpreter.eval_batch with pinned host buffers at several
pipelining chunk sizes.  python tools/e2e_probe.py [n]"""
import sys
import time

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2102_08514_b200.runtime import PlanInterpreter  # noqa: E402


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps, (time.perf_counter() - t0) * 1e3 / reps


def main():
    n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 100_000_000
    dev = torch.device("cuda", 0)
    _, grid, pts, interp = bench.make_workload("tricubic_cc256_fp32", 0, dev, n_override=n)
    hp = pts.cpu().pin_memory()
    ho = torch.empty(n, dtype=grid.dtype).pin_memory()
    dout = torch.empty(n, dtype=grid.dtype, device=dev)
    print("H2D pts  ms (event, wall):", timed(lambda: pts.copy_(hp, non_blocking=True)))
    print("D2H out  ms:", timed(lambda: ho.copy_(dout, non_blocking=True)))
    s2 = torch.cuda.Stream()

    def both():
        cur = torch.cuda.current_stream()
        s2.wait_stream(cur)
        pts.copy_(hp, non_blocking=True)
        with torch.cuda.stream(s2):
            ho.copy_(dout, non_blocking=True)
        cur.wait_stream(s2)

    print("H2D+D2H concurrent ms:", timed(both))
    for chunk in (1 << 30, 1 << 25, 1 << 24, 1 << 23, 1 << 22):
        interp.host_chunk = chunk
        ms = timed(lambda: interp.eval_batch(grid, hp, out=ho, check=False, order="morton"))
        print(f"eval_batch host chunk={chunk}: ms (event, wall) {ms}  -> {n / ms[0] / 1e6:.2f} Gpts/s")


if __name__ == "__main__":
    main()
