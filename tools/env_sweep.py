"""Time one bench workload (protocol A, prepared brick batch) under several SP_* environment
settings in one process: the kernels read their knobs per call.

    python tools/env_sweep.py --workload tricubic_cc256_fp32 --iters 20 \
        "SP_UNITS=0" "SP_UNIT_P=2" "SP_UNIT_P=3" "SP_UNIT_P=4"
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
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("settings", nargs="*", default=[""])
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    plan, grid, pts, interp = bench.make_workload(a.workload, 0, dev, order="morton", n_override=a.points)
    out = torch.empty(pts.shape[0], dtype=grid.dtype, device=dev)
    batch = interp.prepare(grid, pts, presorted=True)
    ref = None
    for rnd in range(2):
        for s in a.settings:
            env = dict(kv.split("=", 1) for kv in s.split(",") if kv)
            old = {k: os.environ.get(k) for k in env}
            os.environ.update(env)
            for _ in range(3):
                interp.eval_batch(grid, batch, out=out, check=False)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(a.iters):
                interp.eval_batch(grid, batch, out=out, check=False)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / a.iters
            if ref is None:
                ref = out.clone()
                same = True
            else:
                same = bool(torch.equal(torch.nan_to_num(out), torch.nan_to_num(ref)))
            n = out.shape[0]
            print(f"round {rnd} {a.workload} [{s or 'default'}] {ms:.3f} ms {n / ms / 1e6:.2f} Gpts/s "
                  f"bit-identical-to-first={same}", flush=True)
            for k, v in old.items():
                if v is None:
                    os.environ.pop(k, None)
                else:
                    os.environ[k] = v


if __name__ == "__main__":
    main()
