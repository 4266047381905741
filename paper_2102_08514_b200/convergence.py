"""Function-approximation (convergence) harness — SURVEY.md §8f rank 3.

`run_convergence(plan, target, prefilter, halvings, samples)` measures the approximation
order of a spline on its lattice the way the paper's §5.2 study does: at each scale h the
target is sampled at the scaled lattice sites f(h·L·n), optionally convolved with the
quasi-interpolation prefilter (`prefilter.apply_prefilter`, the reference's taps), then
reconstructed at Monte-Carlo points x of a centred box with
`PlanInterpreter.eval_batch(grid, x / h)`, and the L2 error is recorded; the fitted order is
the least-squares slope of log2(error) against -log2(h).  Everything after the choice of
points runs on the GPU through the same kernels as the benchmark (one evaluation of
`samples` points per scale), so the harness doubles as an at-scale correctness check of
the reconstruction: a wrong weight, class or fetch shows up as a wrong order.

The reference does not ship this harness (SPEC.md:508-516 describes it); its expected
outcomes are the spline orders of the paper's Table 1 (`corpus.REFERENCE_ORDERS`) and
partition of unity for constant targets.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Callable, Mapping

import numpy as np
import torch

from .prefilter import apply_prefilter
from .runtime import CoefficientGrid, PlanInterpreter

Target = Callable[[torch.Tensor], torch.Tensor]  # (m, 3) float64 positions -> (m,) values


def gaussian(center=(0.05, -0.03, 0.02), sigma: float = 0.25) -> Target:
    """SPEC.md:514 target: exp(-|x - c|^2 / (2 sigma^2)) (the centre truncated to the
    points' dimension)."""
    c = torch.tensor(center, dtype=torch.float64)

    def f(x: torch.Tensor) -> torch.Tensor:
        d = x - c[: x.shape[1]].to(x.device)
        return torch.exp(-(d * d).sum(-1) / (2.0 * sigma * sigma))

    return f


def constant(value: float = 1.0) -> Target:
    def f(x: torch.Tensor) -> torch.Tensor:
        return torch.full((x.shape[0],), value, dtype=torch.float64, device=x.device)

    return f


@dataclass
class ConvergenceReport:
    plan: str
    scales: list = field(default_factory=list)  # h per level
    errors: list = field(default_factory=list)  # RMS error per level
    max_errors: list = field(default_factory=list)
    fitted_order: float = float("nan")
    prefiltered: bool = False


def _fit_order(hs, errs) -> float:
    x = -np.log2(np.asarray(hs, dtype=np.float64))
    y = np.log2(np.maximum(np.asarray(errs, dtype=np.float64), 1e-300))
    a = np.vstack([x, np.ones_like(x)]).T
    slope = np.linalg.lstsq(a, y, rcond=None)[0][0]
    return float(-slope)


def sample_grid(cosets, target: Target, h: float, box: float, margin: int, *, device, dtype,
                boundary: str = "zero") -> CoefficientGrid:
    """Coefficient grid of f(h * site) over all lattice sites within box/h + margin."""
    r = int(math.ceil(box / h)) + margin
    s = len(cosets.diag)
    grid = CoefficientGrid.zeros(cosets, [-r] * s, [r] * s, boundary=boundary, device=device, dtype=dtype)
    diag = torch.tensor(cosets.diag, dtype=torch.float64, device=device)
    for k, arr in enumerate(grid.arrays):
        axes = [torch.arange(n, device=device, dtype=torch.float64) + o for n, o in zip(arr.shape, grid.origins[k])]
        z = torch.stack(torch.meshgrid(*axes, indexing="ij"), -1).reshape(-1, s)
        site = z * diag + torch.tensor(cosets.shifts[k], dtype=torch.float64, device=device)
        arr.copy_(target(h * site).reshape(arr.shape).to(dtype))
    return grid


def spline_center(plan) -> tuple:
    """Centroid of the (non-centred) box spline = half the sum of its
    direction vectors: sum_m c_m phi(y - m) with c_m = f(h m) approximates f(h (y - centre))."""
    from .corpus import direction_set

    cols = direction_set(plan.name.replace("_ungrouped", ""))[0]
    return tuple(sum(c[i] for c in cols) / 2.0 for i in range(len(cols[0])))


def run_convergence(plan, target: Target, *, prefilter: Mapping | None = None, h0: float = 0.25,
                    halvings: int = 4, samples: int = 1_000_000, box: float = 0.5, seed: int = 0,
                    dtype: torch.dtype = torch.float64, device=None) -> ConvergenceReport:
    """SPEC.md:508-516.  Scales h0 / 2^i for i < halvings; Monte-Carlo points uniform in the
    centred box [-box, box]^s; the grid covers the box plus the spline's support."""
    from .lattice import decompose_cartesian, named_lattice

    device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    cos = decompose_cartesian(named_lattice(plan.lattice_name))
    interp = PlanInterpreter(plan)
    gen = torch.Generator(device=device).manual_seed(seed)
    x = (torch.rand((samples, plan.s), generator=gen, device=device, dtype=torch.float64) * 2.0 - 1.0) * box
    fx = target(x)
    rep = ConvergenceReport(plan=plan.name, prefiltered=prefilter is not None)
    margin = 8 + max(cos.diag)  # covers every corpus spline's support (SURVEY.md §9 footprints)
    center = spline_center(plan)
    for i in range(halvings):
        h = h0 / (2 ** i)
        grid = sample_grid(cos, target, h, box, margin, device=device, dtype=dtype)
        if prefilter is not None:
            grid = apply_prefilter(grid, prefilter)
        y = x / h + torch.tensor(center, dtype=torch.float64, device=device)
        if plan.s == 3:  # norms need no caller order: values in brick order + permutation
            s, perm = interp.eval_batch_unordered(grid, y.to(dtype))
            err = s.to(torch.float64) - fx[perm]
        else:
            err = interp.eval_batch(grid, y.to(dtype), order="sort").to(torch.float64) - fx
        rep.scales.append(h)
        rep.errors.append(float(torch.sqrt((err * err).mean())))
        rep.max_errors.append(float(err.abs().max()))
    rep.fitted_order = _fit_order(rep.scales, rep.errors)
    return rep
