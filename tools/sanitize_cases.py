"""Small invocations of every kernel family with cross-path parity checks — a stand-in for
the compute-sanitizer runs SURVEY.md §5's race-detection row suggests (compute-sanitizer is
closed on this pool).  With SP_DEBUG_CHECKS-style bounds checks absent, the checks here are:
every path bit-identical to the chunk kernel, under CUDA_LAUNCH_BLOCKING=1 as well.

    python tools/sanitize_cases.py [--quick]

Paths covered: chunk kernel (order='given'), brick kernel (generic staging, TMA staging,
signature grouping, affine tables), protocol B (indirect and gathered), the fp64 paths, the
texture variant, the prefilter (TMA planes and cp.async) and the ray-marcher.  Each case
also checks its values against the chunk kernel so a sanitizer run is a parity run too.
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2102_08514_b200 import corpus  # noqa: E402
from paper_2102_08514_b200.plan import PlanOptions  # noqa: E402
from paper_2102_08514_b200.runtime import CoefficientGrid, PlanInterpreter  # noqa: E402

PLANS = ["cc_trilinear", "cc_tricubic", "bcc_linear_rd", "bcc_quintic_rd", "fcc_cubic", "cc_zp3", "bcc_quartic",
         "fcc_voronoi1", "bcc_voronoi1"]


def grid_for(name, hi, boundary, dtype, dev, seed):
    _, cos = corpus.lattice_of(name)
    grid = CoefficientGrid.zeros(cos, [0, 0, 0], [hi, hi, hi], boundary=boundary, device=dev, dtype=dtype)
    gen = torch.Generator(device=dev).manual_seed(seed)
    for a in grid.arrays:
        a.copy_(torch.rand(a.shape, generator=gen, device=dev, dtype=dtype))
    return grid


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true", help="fewer points / plans (racecheck is slow)")
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    n = 3000 if a.quick else 20000
    hi = 23
    rng = np.random.default_rng(5)
    cases = 0
    for name in PLANS if not a.quick else ["cc_tricubic", "bcc_linear_rd", "fcc_cubic"]:
        plan = corpus.build_plan(name, PlanOptions(grouped=False)) if name == "cc_zp3" else corpus.build_plan(name)
        interp = PlanInterpreter(plan)
        for dtype in (torch.float32, torch.float64):
            for boundary in ("zero", "mirror"):
                grid = grid_for(name, hi, boundary, dtype, dev, cases)
                pts = torch.from_numpy(rng.uniform(-2, hi + 2, size=(n, 3))).to(dev, dtype)
                want = interp.eval_batch(grid, pts, order="given")
                batch = interp.prepare(grid, pts)
                # brick kernel over the sorted batch, results scattered back to the caller's order
                torch.testing.assert_close(interp.eval_batch(grid, batch), want, rtol=0, atol=0)
                for gather in (False, True):
                    interp.sort_gather = gather
                    torch.testing.assert_close(interp.eval_batch(grid, pts, order="sort"), want, rtol=0, atol=0)
                interp.sort_gather = False
                # protocol B with the result scatter as a separate pass (both variants)
                interp.scatter_window = 1024
                for sorted_scatter in (True, False):
                    interp.scatter_sorted = sorted_scatter
                    torch.testing.assert_close(interp.eval_batch(grid, pts, order="sort"), want, rtol=0, atol=0)
                vals, perm = interp.eval_batch_unordered(grid, pts)
                torch.testing.assert_close(vals, want[perm.long()], rtol=0, atol=0)
                interp.scatter_window = type(interp).scatter_window
                interp.scatter_sorted = True
                cases += 1
                print(f"ok {name} {str(dtype)[6:]} {boundary} ({interp.kernel_name()})", flush=True)
        if name in ("cc_tricubic", "bcc_linear_rd"):
            grid = grid_for(name, hi, "zero", torch.float32, dev, 99)
            pts = torch.from_numpy(rng.uniform(0, hi, size=(n, 3))).to(dev, torch.float32)
            interp.eval_batch_texture(grid, pts)
            print(f"ok {name} texture", flush=True)

    from paper_2102_08514_b200.prefilter import apply_prefilter

    for boundary in ("zero", "clamp"):
        for hi2 in (63, 61):  # 16-byte rows (TMA planes) / odd rows (cp.async)
            _, cos = corpus.lattice_of("bcc_quintic_rd")
            grid = CoefficientGrid.zeros(cos, [0, 0, 0], [21, 19, hi2], boundary=boundary, device=dev)
            for k, arr in enumerate(grid.arrays):
                arr.copy_(torch.rand(arr.shape, device=dev))
            apply_prefilter(grid, corpus.prefilter_taps("bcc_quintic_rd"))
            print(f"ok prefilter {boundary} hi2={hi2}", flush=True)

    from paper_2102_08514_b200.render import Camera, RenderJob, ml_volume, render_volume

    plan = corpus.build_plan("bcc_linear_rd")
    grid, sc, off = ml_volume(plan, 12, device=dev)
    job = RenderJob(plan=plan, volume=grid, width=12, height=10, n_steps=24, step=0.08, lattice_scale=sc,
                    lattice_offset=off, slab=12, camera=Camera(position=(0.1, -0.05, -1.4), fov=2.4))
    render_volume(job)
    torch.cuda.synchronize()
    print(f"ok render; {cases} eval cases", flush=True)


if __name__ == "__main__":
    main()
