#!/usr/bin/env python
"""Benchmark: Gpoints/s reconstructed on B200 (BASELINE.json metric) + roofline + CPU baseline.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...          (one rank per GPU, NCCL)

Headline workload (BASELINE.json configs[1]): tricubic tensor-product
B-spline on a CC 256^3 lattice, 10^8 uniformly random query points per GPU, fp32,
boundary 'zero'.  A step = one `PlanInterpreter.eval_batch` over the whole batch (one
kernel launch), inputs resident in HBM.  Input-order protocol (A) of SURVEY.md §8d: the
iid-uniform points are presented in Morton (Z-curve) order of their unit cell, generated
once outside the timed region; protocol (B) — the same points shuffled, evaluated
through the `reorder=True` path that Morton-sorts on the GPU inside the timed region —
is reported as `unsorted_e2e_device`.  Points (1.2 GB) exceed L2, so no flush is needed.

Other BASELINE configs are measured in the same run under "workloads" (parity for all of
them is in tests/).  `e2e` is the same metric through the public API with pinned HOST
buffers: H2D points + kernel + D2H results per step.

`--impl reference` times the reference CPU algorithm (the numpy restatement in
oracle/plan_numpy.py of runtime.py:363-408, all host cores via fork) on a bounded sample
of the same workload.
"""

from __future__ import annotations

import argparse
import json
import math
import multiprocessing as mp
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Gpoints/s reconstructed (CC/BCC/FCC, 1/2/4/8 B200) and % of memory roofline"
UNIT = "Gpoints/s"

# name -> (plan, grid hi (lo=0), dtype, points per GPU)
WORKLOADS = {
    "tricubic_cc256_fp32": ("cc_tricubic", 255, "float32", 100_000_000),
    "tricubic_cc256_fp64": ("cc_tricubic", 255, "float64", 100_000_000),
    "trilinear_cc64_fp32": ("cc_trilinear", 63, "float32", 1_000_000),
    "bcc_linear_2x203_fp32": ("bcc_linear_rd", 405, "float32", 100_000_000),
    "bcc_quintic_2x203_fp32": ("bcc_quintic_rd", 405, "float32", 100_000_000),
    "fcc6_4x161_fp32": ("fcc_cubic", 321, "float32", 100_000_000),
    "zp3_cc256_fp32": ("cc_zp3", 255, "float32", 100_000_000),
    # float64 (the reference's only precision, runtime.py:57, :248) for C3/C4
    "bcc_linear_2x203_fp64": ("bcc_linear_rd", 405, "float64", 100_000_000),
    "bcc_quintic_2x203_fp64": ("bcc_quintic_rd", 405, "float64", 100_000_000),
    "fcc6_4x161_fp64": ("fcc_cubic", 321, "float64", 100_000_000),
    "zp3_cc256_fp64": ("cc_zp3", 255, "float64", 100_000_000),
    # C5: Voronoi splines V1 at 512^3-equivalent samples (BCC 2x406^3, FCC 4x322^3), 10^9 points
    # per GPU.  PP data: tools/voronoi_pp.py (reference exact tools), plans: reference compiler.
    "c5_fcc_voronoi1_4x322_1e9_fp32": ("fcc_voronoi1", 643, "float32", 1_000_000_000),
    "c5_bcc_voronoi1_2x406_1e9_fp32": ("bcc_voronoi1", 811, "float32", 1_000_000_000),
    # the BCC linear box spline on the C5 BCC geometry (HBM-bound reference point)
    "bcc_linear_2x406_1e9_fp32": ("bcc_linear_rd", 811, "float32", 1_000_000_000),
}
HEADLINE = "tricubic_cc256_fp32"

_REASONS = {
    0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
    0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
    0x100: "display_clock_setting",
}


def _plan_name(name: str) -> str:
    from paper_2102_08514_b200 import corpus

    plans = corpus.available_plans()
    if name in plans:
        return name
    if f"{name}_ungrouped" in plans:
        return f"{name}_ungrouped"
    raise KeyError(name)


# ---------------------------------------------------------------------------------------
# clocks sampler (NVML, during the timed region)


class ClockSampler:
    def __init__(self, index: int, period_s: float = 0.002):
        self.index = index
        self.period = period_s
        self.samples = []
        self.reasons = 0
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None

    def __enter__(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)

            def run():
                while not self._stop.is_set():
                    try:
                        self.samples.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
                        self.reasons |= pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                    except Exception:
                        pass
                    time.sleep(self.period)

            self._t = threading.Thread(target=run, daemon=True)
            self._t.start()
        except Exception:
            self._t = None
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._t is not None:
            self._t.join(timeout=1)

    def summary(self) -> dict:
        reasons = [name for bit, name in _REASONS.items() if self.reasons & bit]
        return {
            "sm_mhz": float(np.median(self.samples)) if self.samples else None,
            "sm_max_mhz": self.max_mhz,
            "reasons": reasons,
            "samples": len(self.samples),
        }


# ---------------------------------------------------------------------------------------
# workload setup


def make_workload(name, rank, device, order="morton", n_override=None):
    import torch

    from paper_2102_08514_b200 import corpus
    from paper_2102_08514_b200.runtime import CoefficientGrid, PlanInterpreter, morton_order

    plan_name, hi, dt, n = WORKLOADS[name]
    n = n_override or n
    dtype = getattr(torch, dt)
    plan = corpus.load_plan(corpus.PLAN_DIR / f"{_plan_name(plan_name)}.plan.json")
    _, cos = corpus.lattice_of(plan_name)
    grid = CoefficientGrid.zeros(cos, [0, 0, 0], [hi, hi, hi], device=device, dtype=dtype)
    gen = torch.Generator(device=device).manual_seed(2102_08514 + 7919 * rank)
    for a in grid.arrays:  # coefficients uniform in [0,1), generated as fp32
        a.copy_(torch.rand(a.shape, generator=gen, device=device, dtype=torch.float32).to(dtype))
    pts = (torch.rand((n, 3), generator=gen, device=device, dtype=torch.float32) * (hi + 1)).to(dtype)
    if order == "morton":
        perm = morton_order(pts)
        pts = pts[perm].contiguous()
        del perm
    interp = PlanInterpreter(plan)
    return plan, grid, pts, interp


def algorithmic_bytes(n, grid, dtype_size):
    """B/pt = s*sizeof(T_pt) + sizeof(T_out) + lattice/n."""
    return n * (3 * dtype_size + dtype_size) + grid.nbytes()


def onchip_roofline(plan, esize, pts_per_s, sm_mhz):
    """Secondary (on-chip) roofline, SURVEY.md §8d 'secondary bounds': the tensor-product
    kernels are bound by the shared-memory datapath (every point receives (DEG+1)^3 taps,
    128 B per SM per clock), the box-spline kernels by the FP32 pipe (the plan's weight
    programs, 128 FMA lanes per SM per clock).  Peaks at the clock sampled during the run."""
    from paper_2102_08514_b200 import codegen

    clk = (sm_mhz or 1965.0) * 1e6
    deg = plan.tensor_bspline_degree()
    if deg is not None:
        taps = (deg + 1) ** 3
        per_pt = taps * esize
        peak = 148 * 128 * clk
        return {"bound": "shared-memory datapath", "unit": "TB/s", "bytes_per_point": per_pt,
                "achieved": pts_per_s * per_pt / 1e12, "peak": peak / 1e12, "frac": pts_per_s * per_pt / peak}
    if not codegen.codegen_supported(plan):
        return None
    fl = codegen.weight_flops(plan)
    per_pt = plan.M * sum(fl) / len(fl)  # specialised (one kernel per coset), mean over kernels
    # B200: 128 FP32 FMA lanes per SM per clock; FP64 at half rate (datasheet 40 vs 80 TFLOPS)
    peak = 148 * 128 * clk * (1.0 if esize == 4 else 0.5)
    return {"bound": "fp32 pipe (weight programs)" if esize == 4 else "fp64 pipe (half the fp32 rate)",
            "unit": "Top/s (FMA = 1 op)",
            "flops_per_point": per_pt, "flops_per_coset_per_kernel": fl,
            "achieved": pts_per_s * per_pt / 1e12, "peak": peak / 1e12, "frac": pts_per_s * per_pt / peak}


def bench_prefilter(args, device, rank, stream, dist, peak, hi=811):
    """the quasi-interpolation prefilter of the BCC quintic spline
    (9 taps, corpus.py:71-82) over the C5 grid (BCC 2x406^3, fp32, 535 MB > L2).  Streaming
    stencil: algorithmic HBM bytes = one read + one write of every coset sample."""
    import torch

    from paper_2102_08514_b200 import corpus
    from paper_2102_08514_b200.prefilter import apply_prefilter
    from paper_2102_08514_b200.runtime import CoefficientGrid

    _, cos = corpus.lattice_of("bcc_quintic_rd")
    grid = CoefficientGrid.zeros(cos, [0, 0, 0], [hi, hi, hi], device=device, dtype=torch.float32)
    gen = torch.Generator(device=device).manual_seed(2102_08514 + 31 * rank)
    for a in grid.arrays:
        a.copy_(torch.rand(a.shape, generator=gen, device=device))
    taps = corpus.prefilter_taps("bcc_quintic_rd")
    out = apply_prefilter(grid, taps)
    ms = measure(lambda: apply_prefilter(grid, taps, out=out), max(3, min(args.steps, 50)), args.warmup, stream, dist)
    nbytes = 2 * grid.nbytes()
    gbs = nbytes / (ms * 1e-3) / 1e9
    n = (hi + 1) // 2
    return {"workload": f"bcc_quintic_rd prefilter (9 taps) on BCC 2x{n}^3 fp32, zero policy",
            "staging": "TMA planes (16-byte coset rows)" if (n * 4) % 16 == 0 else "cp.async (rows not 16-byte multiples)",
            "value": gbs, "unit": "GB/s", "ms_per_step": ms, "samples": grid.site_count(),
            "algorithmic_bytes_per_step": nbytes, "roofline_hbm_frac": gbs / peak,
            "l2": f"input and output {grid.nbytes() / 1e6:.0f} MB each > 126 MB L2"}


def bench_render(args, device):
    """the ray-marcher consuming reconstruction (render.py,
    SPEC.md render_volume).  Marschner-Lobb on CC 128^3 sampled for the tricubic spline,
    512x512 orthographic view, 384 steps of 1/128: 100.7 M reconstructions per frame plus
    compositing.  Best of a few frames after a warm-up frame (CUDA events)."""
    import torch

    from paper_2102_08514_b200 import corpus
    from paper_2102_08514_b200.render import Camera, RenderJob, ml_volume, render_volume
    from paper_2102_08514_b200.runtime import PlanInterpreter

    plan = corpus.build_plan("cc_tricubic")
    grid, sc, off = ml_volume(plan, 128, device=device)
    job = RenderJob(plan=plan, volume=grid, width=512, height=512, n_steps=384, step=1.0 / 128, lattice_scale=sc,
                    lattice_offset=off, slab=64, camera=Camera(position=(0.0, 0.0, -1.5), fov=2.2))
    interp = PlanInterpreter(plan)
    render_volume(job, interp)
    ms = min(render_volume(job, interp).ms for _ in range(3))
    samples = job.width * job.height * job.n_steps
    return {"workload": "Marschner-Lobb (f_M=6, alpha=0.25) on CC 128^3, cc_tricubic, 512x512, 384 steps, fp32",
            "ms_per_frame": ms, "value": samples / (ms * 1e-3) / 1e9, "unit": "Gsamples/s (reconstruct + composite)",
            "samples_per_frame": samples}


def measure(fn, steps, warmup, stream, dist=None):
    import torch

    for _ in range(warmup):
        fn()
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    start = torch.cuda.Event(enable_timing=True)
    end = torch.cuda.Event(enable_timing=True)
    start.record(stream)
    for _ in range(steps):
        fn()
    end.record(stream)
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    ms = start.elapsed_time(end) / steps
    if dist is not None:
        t = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    return ms


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def load_traffic(name):
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(path):
        with open(path) as fh:
            d = json.load(fh)
        v = d.get(name)
        if isinstance(v, dict):
            return v.get("dram_bytes_per_launch")
        return v
    return None


# ---------------------------------------------------------------------------------------
# CPU arm: numpy restatement of the reference batch path (oracle/, checker only)

_CPU_STATE = {}


def _cpu_chunk(args):
    lo, hi = args
    from oracle.plan_numpy import eval_batch

    st = _CPU_STATE
    return eval_batch(st["plan"], st["grid"], st["pts"][lo:hi], st["tabs"])


def cpu_reference_setup(name, seed=0):
    """Host grid + a point pool for the CPU arm (same distribution as the GPU workload)."""
    from oracle.plan_numpy import NumpyGrid, PlanTables
    from paper_2102_08514_b200 import corpus
    from paper_2102_08514_b200.runtime import grid_extents

    plan_name, hi, _, _ = WORKLOADS[name]
    plan = corpus.load_plan(corpus.PLAN_DIR / f"{_plan_name(plan_name)}.plan.json")
    _, cos = corpus.lattice_of(plan_name)
    origins, shapes = grid_extents(cos, [0, 0, 0], [hi, hi, hi])
    rng = np.random.default_rng(2102_08514 + seed)
    arrays = [rng.random(sh, dtype=np.float32).astype(np.float64) for sh in shapes]
    pts = (rng.random((1 << 20, 3), dtype=np.float32) * np.float32(hi + 1)).astype(np.float64)
    _CPU_STATE.update(plan=plan, grid=NumpyGrid(plan.diag, plan.shifts, arrays, origins, "zero"), pts=pts,
                      tabs=PlanTables(plan))


def cpu_run(n_points, pool, chunk=2048):
    spans = [(i, min(i + chunk, n_points)) for i in range(0, n_points, chunk)]
    t0 = time.perf_counter()
    if pool is None:
        for s in spans:
            _cpu_chunk(s)
    else:
        pool.map(_cpu_chunk, spans)
    return time.perf_counter() - t0


def cpu_calibrated_sample(pool, cores, target_s):
    """Points per sample so that one sample takes ~target_s on `cores` workers."""
    t = cpu_run(1024, None, chunk=1024)  # one core, includes first-touch costs
    t = cpu_run(1024, None, chunk=1024)
    rate = 1024 / max(t, 1e-6)  # pts/s/core
    n = int(rate * cores * target_s)
    n = max(2048, min(n, len(_CPU_STATE["pts"])))
    return (n // 2048) * 2048 or 2048


def cpu_baseline(name, budget_s=15.0):
    cpu_reference_setup(name)
    cores = os.cpu_count() or 1
    ctx = mp.get_context("fork")
    with ctx.Pool(cores) as pool:
        n = cpu_calibrated_sample(pool, cores, budget_s)
        secs = cpu_run(n, pool)
    return {
        "value": n / secs / 1e9,
        "unit": UNIT,
        "cores": cores,
        "kind": "port",
        "sample": f"{n} uniform points of {name} (same grid shape/distribution), numpy restatement of "
                  f"runtime.py:363-408 (oracle/plan_numpy.py), fp64, {cores} fork workers, {secs:.1f} s",
        "seconds": secs,
    }


# ---------------------------------------------------------------------------------------
# CPU arm: the REFERENCE itself (splineplan installed into baseline/_ref, PlanInterpreter.
# eval_batch, runtime.py:244-248) on the host cores; the numpy port (oracle/) when the
# install is absent.

_REF_STATE = {}
REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def reference_available() -> bool:
    return os.path.isdir(os.path.join(REF_DIR, "splineplan"))


def _ref_chunk(span):
    lo, hi = span
    st = _REF_STATE
    return st["interp"].eval_batch(st["grid"], st["pts"][lo:hi])


def ref_setup(name, seed=0):
    """The reference's own grid / plan / interpreter for a workload (host, float64), the
    same grid shape and point distribution as the GPU workload; state inherited by fork."""
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    from splineplan.lattice import decompose_cartesian, named_lattice
    from splineplan.plancompile import deserialize_plan
    from splineplan.runtime import CoefficientGrid, PlanInterpreter

    from paper_2102_08514_b200 import corpus

    plan_name, hi, _, _ = WORKLOADS[name]
    with open(corpus.PLAN_DIR / f"{_plan_name(plan_name)}.plan.json") as fh:
        plan = deserialize_plan(fh.read())
    cos = decompose_cartesian(named_lattice(plan.lattice_name))
    grid = CoefficientGrid.zeros(cos, [0, 0, 0], [hi, hi, hi])  # runtime.py:65-78
    rng = np.random.default_rng(2102_08514 + seed)
    for a in grid.arrays:
        a[...] = rng.random(a.shape, dtype=np.float32)
    pts = (rng.random((1 << 20, 3), dtype=np.float32) * np.float32(hi + 1)).astype(np.float64)
    interp = PlanInterpreter(plan)
    interp._batch_tables()  # lowered tables built once, before the fork
    _REF_STATE.clear()
    _REF_STATE.update(interp=interp, grid=grid, pts=pts)


REF_CHUNK = 8192


def ref_run(n_points, pool, chunk=REF_CHUNK):
    """Chunks of REF_CHUNK points over the pool (chunking is mandatory,
    _poly_batch allocates n x terms x s); the calibration uses the same chunk size."""
    spans = [(i, min(i + chunk, n_points)) for i in range(0, n_points, chunk)]
    t0 = time.perf_counter()
    if pool is None:
        for sp in spans:
            _ref_chunk(sp)
    else:
        pool.map(_ref_chunk, spans)
    return time.perf_counter() - t0


def ref_calibrated_sample(cores, target_s, pool=None):
    """Points per sample so that one pooled sample takes ~target_s (calibrated on the pool
    itself: memory-bound numpy scales sub-linearly with the worker count)."""
    ref_run(256, None)  # first-touch costs
    n0 = min(REF_CHUNK * cores, len(_REF_STATE["pts"]))
    t = ref_run(n0, pool)
    n = int(n0 / max(t, 1e-6) * target_s)
    return max(256 * cores, min(n, len(_REF_STATE["pts"])))


def cpu_baseline_reference(name, budget_s):
    """cpu_baseline of one workload with the reference's own eval_batch (all host cores)."""
    ref_setup(name)
    cores = os.cpu_count() or 1
    with mp.get_context("fork").Pool(cores) as pool:
        n = ref_calibrated_sample(cores, budget_s, pool)
        secs = ref_run(n, pool)
    _REF_STATE.clear()
    return {"value": n / secs / 1e9, "unit": UNIT, "cores": cores, "kind": "reference",
            "sample": f"{n} uniform points of {name} (same grid shape/distribution), splineplan "
                      f"PlanInterpreter.eval_batch from baseline/_ref (runtime.py:244-248), float64, chunks of "
                      f"8192 points over {cores} fork workers, {secs:.1f} s", "seconds": secs}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    name = args.workload
    cores = os.cpu_count() or 1
    step_s = min(args.ref_step_seconds, args.ref_total_seconds / max(1, args.steps + args.warmup))
    port = None
    if reference_available():
        kind = "reference"
        ref_setup(name)
        with mp.get_context("fork").Pool(cores) as pool:
            n = ref_calibrated_sample(cores, step_s, pool)
            for _ in range(args.warmup):
                ref_run(n, pool)
            times = [ref_run(n, pool) for _ in range(args.steps)]
        _REF_STATE.clear()
        sample = (f"{n} uniform points per step, splineplan PlanInterpreter.eval_batch from baseline/_ref "
                  f"(runtime.py:244-248, the unmodified reference), float64, chunks of 8192 points over "
                  f"{cores} fork workers")
        # the numpy port of the same algorithm (oracle/plan_numpy.py), for comparison
        try:
            port = cpu_baseline(name, min(5.0, step_s))
        except Exception as exc:  # noqa: BLE001
            port = {"unavailable": repr(exc)}
    else:
        kind = "port"
        cpu_reference_setup(name)
        with mp.get_context("fork").Pool(cores) as pool:
            n = cpu_calibrated_sample(pool, cores, step_s)
            for _ in range(args.warmup):
                cpu_run(n, pool)
            times = [cpu_run(n, pool) for _ in range(args.steps)]
        sample = (f"{n} uniform points per step, numpy restatement of runtime.py:363-408 "
                  f"(oracle/plan_numpy.py; baseline/_ref not installed), {cores} fork workers")
    secs = float(np.mean(times))
    value = n / secs / 1e9
    plan_name, hi, _, _ = WORKLOADS[name]
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": secs * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": name, "points_per_step": n, "grid_hi": hi, "spline": plan_name, "boundary": "zero"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": kind, "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    if port is not None:
        line["port_baseline"] = port
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------------------
# GPU arm


def bench_c5_strong(args, device, rank, world, stream, dist, wname):
    """C5 as north_star states it (BASELINE.json configs[4]): 10^9 points in
    TOTAL sharded n/G over the G ranks (each rank generates its own shard, Morton-ordered as
    protocol A), lattice replicated; per-rank evaluation time max-reduced over ranks; then, for a
    caller who wants ONE output tensor, the all-gather of the shards over NCCL
    (sharding.gather_results), timed separately."""
    import torch

    from paper_2102_08514_b200.sharding import gather_results, shard_range

    total = WORKLOADS[wname][3]
    a, b = shard_range(total, rank, world)
    nloc = b - a
    plan, grid, pts, interp = make_workload(wname, rank, device, n_override=nloc)
    batch = interp.prepare(grid, pts, presorted=True)
    out = torch.empty(nloc, dtype=grid.dtype, device=device)

    def step():
        interp.eval_batch(grid, batch, out=out, check=False)

    step()
    torch.cuda.synchronize()
    steps = max(3, min(args.steps, 10))
    ms = measure(step, steps, args.warmup, stream, dist)
    gather_ms = 0.0
    if dist is not None:
        width = max(y - x for x, y in (shard_range(total, r, world) for r in range(world)))
        full = torch.empty(world * width, dtype=grid.dtype, device=device)
        gather_ms = measure(lambda: gather_results(out, total, out=full), steps, 1, stream, dist)
        del full
    res = {"workload": wname, "spline": WORKLOADS[wname][0], "scaling": "strong", "total_points": total,
           "per_rank_points": nloc, "n_ranks": world, "ms_per_step": ms, "value": total / (ms * 1e-3) / 1e9,
           "gather_ms": gather_ms, "value_with_gather": total / ((ms + gather_ms) * 1e-3) / 1e9, "unit": UNIT,
           "gather": "all_gather_into_tensor of n*4 B over NCCL (NVLink), one output tensor on every rank"
                     if world > 1 else "single rank: the output is already one tensor"}
    del plan, grid, pts, interp, batch, out
    torch.cuda.empty_cache()
    return res


def run_ours(args):
    import torch
    import torch.distributed as torch_dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    dist = None
    if world > 1:
        torch_dist.init_process_group("nccl", device_id=device)
        dist = torch_dist
    peak, peak_kind = load_peaks()
    stream = torch.cuda.current_stream(device)

    from paper_2102_08514_b200 import _native

    # ---- headline -------------------------------------------------------------------
    name = args.workload
    plan, grid, pts, interp = make_workload(name, rank, device, n_override=args.points)
    n = pts.shape[0]
    out = torch.empty(n, dtype=grid.dtype, device=device)
    launches_per_step = _native.lib().sp_eval_launch_count(interp._handle(device), n)

    # protocol A: points presented in Morton order; the brick runs are part of the layout
    batch = interp.prepare(grid, pts, presorted=True)

    def step():
        interp.eval_batch(grid, batch, out=out, check=False)

    step()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        ms = measure(step, args.steps, args.warmup, stream, dist)
    esize = grid.arrays[0].element_size()
    bytes_launch = algorithmic_bytes(n, grid, esize)
    achieved = bytes_launch / (ms * 1e-3) / 1e9
    value = world * n / (ms * 1e-3) / 1e9

    # ---- e2e through the public API with pinned host buffers --------------------------
    host_pts = pts.to("cpu").pin_memory()
    host_out = torch.empty(n, dtype=grid.dtype).pin_memory()

    if args.e2e_chunk:
        interp.host_chunk = args.e2e_chunk

    def e2e_step():
        interp.eval_batch(grid, host_pts, out=host_out, check=False, order="morton")

    e2e_steps = max(2, min(args.steps, args.e2e_steps))
    e2e_ms = measure(e2e_step, e2e_steps, max(1, min(args.warmup, 3)), stream, dist)
    e2e_each = []  # per-step spread (diagnostic; the value above is the K-step mean)
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        e2e_step()
        e1.record(stream)
        torch.cuda.synchronize()
        e2e_each.append(round(e0.elapsed_time(e1), 3))
    e2e = {
        "value": world * n / (e2e_ms * 1e-3) / 1e9, "unit": UNIT,
        "h2d_bytes_per_step": int(host_pts.numel() * host_pts.element_size()),
        "d2h_bytes_per_step": int(host_out.numel() * host_out.element_size()),
        "ms_per_step": e2e_ms, "steps": e2e_steps, "extra_step_ms": e2e_each,
        "path": "PlanInterpreter.eval_batch(grid, pinned CPU tensor, out=pinned CPU tensor, order='morton')",
    }
    del host_pts, host_out

    # ---- the public call on device tensors: eval_batch(grid, pts, order="morton") ------
    # (Morton keys + device brick runs + the brick kernel, all inside the timed region)
    def pub_step():
        interp.eval_batch(grid, pts, out=out, check=False, order="morton")

    pub_step()
    torch.cuda.synchronize()
    ms_pub = measure(pub_step, max(3, min(args.steps, 40)), args.warmup, stream, dist)
    public_device = {"value": world * n / (ms_pub * 1e-3) / 1e9, "unit": UNIT, "ms_per_step": ms_pub,
                     "path": "PlanInterpreter.eval_batch(grid, cuda points, out=..., order='morton'): "
                             "sp_morton_keys + sp_brick_runs (count on the device) + brick kernel, no host sync"}

    # ---- hardware-texture-filtered variant (reported separately, with its error) ------
    texture = None
    try:
        tex_out = torch.empty(n, dtype=torch.float32, device=device)
        pts32 = pts.float()

        def tex_step():
            interp.eval_batch_texture(grid, pts32, out=tex_out)

        tex_step()
        torch.cuda.synchronize()
        ms_t = measure(tex_step, max(3, min(args.steps, 40)), args.warmup, stream, dist)
        interp.eval_batch(grid, batch, out=out, check=False)
        ok = torch.isfinite(out)
        err = ((tex_out[ok] - out[ok].float()).abs().max() / out[ok].abs().max()).item()
        texture = {"value": world * n / (ms_t * 1e-3) / 1e9, "unit": UNIT, "ms_per_step": ms_t,
                   "max_err_rel_to_max_f": err,
                   "note": "tex3D hardware trilinear filtering (9-bit weights), 8 fetches/pt for tricubic; "
                           "NOT within the 1e-5 parity tolerance"}
        del tex_out, pts32
    except NotImplementedError as exc:
        texture = {"unavailable": str(exc)}

    # ---- protocol (B): shuffled points, GPU Morton sort inside the timed region -------
    shuffled = pts[torch.randperm(n, device=device)]

    def unsorted_step():
        interp.eval_batch(grid, shuffled, out=out, check=False, order="sort")

    ms_b = measure(unsorted_step, max(2, min(args.steps // 4, 10)), 1, stream, dist)

    def unordered_step():  # values left in brick order, paired with the permutation
        interp.eval_batch_unordered(grid, shuffled, check=False, stream=stream)

    ms_u = measure(unordered_step, max(2, min(args.steps // 4, 10)), 1, stream, dist)
    del shuffled
    torch.cuda.empty_cache()

    line = {
        "metric": METRIC,
        "value": value,
        "unit": UNIT,
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f32" if esize == 4 else "f64",
        "data": "synthetic",
        "config": {
            "workload": name, "spline": WORKLOADS[name][0], "lattice": "CC3", "grid": [256, 256, 256],
            "points_per_gpu": n, "boundary": "zero", "input_order": "morton (protocol A, SURVEY.md §8d)",
            "l2": "inputs larger than L2 (points %.2f GB > 126 MB); lattice %.0f MB L2-resident"
                  % (n * 3 * esize / 1e9, grid.nbytes() / 1e6),
            "parallelism": f"points sharded, lattice replicated, dp{world}",
            "kernel": interp.kernel_name(device),
        },
        "roofline": {
            "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
            "traffic": load_traffic(name), "peak_source": peak_kind,
            "algorithmic_bytes_per_launch": bytes_launch, "bytes_per_point": bytes_launch / n,
            "kernel_ms": ms,
        },
        "e2e": e2e,
        "public_device_morton": public_device,
        "unsorted_e2e_device": {"value": world * n / (ms_b * 1e-3) / 1e9, "unit": UNIT, "ms_per_step": ms_b,
                                "note": "protocol B: shuffled points; Morton keys + sort + brick runs + eval reading "
                                        "the points through the permutation + scatter to caller order, all "
                                        "timed"},
        "unsorted_unordered_device": {"value": world * n / (ms_u * 1e-3) / 1e9, "unit": UNIT, "ms_per_step": ms_u,
                                      "note": "protocol B for reductions: shuffled points; sort + brick kernel "
                                              "reading through the permutation, values returned in brick order with "
                                              "the permutation (eval_batch_unordered), all timed"},
        "roofline_onchip": onchip_roofline(plan, esize, n / (ms * 1e-3), clk.summary().get("sm_mhz")),
        "texture_variant": texture,
        "gpu_launches": int(args.steps * launches_per_step),
        "clocks": clk.summary(),
    }
    del pts, out, grid, batch
    torch.cuda.empty_cache()

    # ---- other BASELINE configs --------------------------------------------------------
    if not args.headline_only:
        others = {}
        for wname in WORKLOADS:
            if wname == name:
                continue
            try:
                plan_w, grid_w, pts_w, interp_w = make_workload(wname, rank, device)
            except KeyError:
                continue
            nw = pts_w.shape[0]
            out_w = torch.empty(nw, dtype=grid_w.dtype, device=device)
            batch_w = interp_w.prepare(grid_w, pts_w, presorted=True)

            # launch-bound batches (C1: 1e6 points, ~10 us of GPU work) replay a CUDA graph of
            # the same eval_batch call instead of paying the Python/ctypes call each step
            graph_w = interp_w.graph(grid_w, batch_w, out=out_w) if nw <= 10_000_000 else None

            def wstep():
                if graph_w is not None:
                    graph_w.replay()
                else:
                    interp_w.eval_batch(grid_w, batch_w, out=out_w, check=False)

            wstep()
            torch.cuda.synchronize()
            msw = measure(wstep, max(3, min(args.steps, 40)), args.warmup, stream, dist)
            es = grid_w.arrays[0].element_size()
            bw = algorithmic_bytes(nw, grid_w, es)
            tex_w = None
            if wname in ("bcc_linear_2x203_fp32", "bcc_quintic_2x203_fp32", "fcc6_4x161_fp32"):
                # the paper's hardware linear-fetch merge for box splines (one filtered texture
                # fetch per 2-site group): reported separately, with its error vs the exact kernel
                tex_out = interp_w.eval_batch_texture(grid_w, batch_w.pts)
                ms_tex = measure(lambda: interp_w.eval_batch_texture(grid_w, batch_w.pts, out=tex_out),
                                 max(3, min(args.steps, 20)), args.warmup, stream, dist)
                ok = torch.isfinite(out_w)
                tex_w = {"value": world * nw / (ms_tex * 1e-3) / 1e9, "unit": UNIT, "ms_per_step": ms_tex,
                         "max_err_rel_to_max_f": float((tex_out[ok] - out_w[ok]).abs().max() / out_w[ok].abs().max()),
                         "note": "one tex3D linear fetch per 2-site fetch group (9-bit weights); NOT within the 1e-5 tolerance"}
                del tex_out
            others[wname] = {
                "value": world * nw / (msw * 1e-3) / 1e9, "unit": UNIT, "ms_per_step": msw,
                "texture_variant": tex_w,
                "points_per_gpu": nw, "kernel": interp_w.kernel_name(device), "cuda_graph": graph_w is not None,
                "roofline_hbm_frac": bw / (msw * 1e-3) / 1e9 / peak, "bytes_per_point": bw / nw,
                "roofline_onchip": onchip_roofline(plan_w, es, nw / (msw * 1e-3), None),
            }
            del plan_w, grid_w, pts_w, interp_w, out_w, batch_w, graph_w
            torch.cuda.empty_cache()
        line["workloads"] = others
        line["prefilter"] = bench_prefilter(args, device, rank, stream, dist, peak)
        line["prefilter_tma"] = bench_prefilter(args, device, rank, stream, dist, peak, hi=1023)
        line["render"] = bench_render(args, device)

    # ---- C5 as north_star states it: 10^9 points in total over the G ranks ------------
    if not args.headline_only:
        line["c5_strong"] = [bench_c5_strong(args, device, rank, world, stream, dist, w)
                             for w in ("c5_fcc_voronoi1_4x322_1e9_fp32", "c5_bcc_voronoi1_2x406_1e9_fp32")]

    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        # the reference itself (baseline/_ref) on the host cores: the headline config and,
        # bounded, every other workload; the numpy port beside it for the headline
        if reference_available():
            line["cpu_baseline"] = cpu_baseline_reference(name, args.cpu_seconds)
            line["cpu_baseline_port"] = cpu_baseline(name, min(args.cpu_seconds, 5.0))
            for wname, w in line.get("workloads", {}).items():
                try:
                    w["cpu_baseline"] = cpu_baseline_reference(wname, args.cpu_seconds_per_workload)
                except Exception as exc:  # noqa: BLE001
                    w["cpu_baseline"] = {"unavailable": repr(exc)}
        else:
            line["cpu_baseline"] = cpu_baseline(name, args.cpu_seconds)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", default=HEADLINE, choices=sorted(WORKLOADS))
    ap.add_argument("--points", type=int, default=None, help="points per GPU (default: the workload's)")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--e2e-chunk", type=int, default=0, help="points per pipelined host chunk (0 = library default)")
    ap.add_argument("--headline-only", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--cpu-seconds-per-workload", type=float, default=3.0)
    ap.add_argument("--ref-step-seconds", type=float, default=4.0)
    ap.add_argument("--ref-total-seconds", type=float, default=150.0,
                    help="time budget of the whole --impl reference run (steps + warmup)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
