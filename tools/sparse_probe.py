import sys, torch
sys.path.insert(0, ".")
import bench
from paper_2102_08514_b200.runtime import prepare_points
dev = torch.device("cuda", 0)
for name in ("tricubic_cc256_fp32", "fcc6_4x161_fp32", "bcc_quintic_2x203_fp32"):
    for n in (1_000_000, 10_000_000, 100_000_000):
        _, grid, pts, interp = bench.make_workload(name, 0, dev, n_override=n)
        out = torch.empty(n, dtype=grid.dtype, device=dev)
        st = torch.cuda.current_stream(dev)
        res = {}
        res["given"] = bench.measure(lambda: interp.eval_batch(grid, pts, out=out, check=False), 20, 3, st)
        bmax = interp.brick_log2(grid)
        for b in range(1, bmax + 1):
            batch = prepare_points(pts, b, presorted=True)
            res[f"b{b}"] = bench.measure(lambda: interp.eval_batch(grid, batch, out=out, check=False), 20, 3, st)
        print(name, n, {k: round(n / v / 1e6, 1) for k, v in res.items()}, "Gpts/s", flush=True)
        del grid, pts, out
        torch.cuda.empty_cache()
