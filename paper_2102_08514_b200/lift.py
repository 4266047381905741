"""Two-dimensional plans on the three-dimensional kernels (the reference corpus' tp2, zp and
qc_tensor splines, corpus.py:35-44).

A plan of dimension s = 2 is evaluated as the s = 3 plan of the same spline times the
degree-0 B-spline (the indicator of [0, 1)) along a third axis: lattice L (+) [1], diagonal
(d0, d1, 1), coset shifts (l, 0), cut planes with a zero third normal component, class
transforms T (+) 1 and pi (+) 1, kernel sites (m, 0) and weight polynomials independent of
y2.  Every point (x0, x1) is evaluated at (x0, x1, 0) over the grid viewed as (n0, n1, 1)
arrays: its coset frame along the new axis is xp2 = 0, cell 0, no plane reads it and no
weight depends on it, so the classification, the sites and the sum are exactly those of
Algorithm 1 in 2-D (runtime.py:363-408) — the same floating-point operations on the same
values.  The views share storage with the caller's grid.
"""

from __future__ import annotations

from fractions import Fraction

import numpy as np
import torch

from .exact import Poly
from .lattice import CosetDecomposition, IntegerLattice
from .plan import ClassTransform, EvaluationPlan, FetchGroup, PlanKernel


def _lift_poly(p: Poly) -> Poly:
    return Poly(3, {tuple(e) + (0,): c for e, c in p.terms.items()})


def lift_plan(plan: EvaluationPlan) -> EvaluationPlan:
    if plan.s != 2:
        raise ValueError("lift_plan lifts s == 2 plans")
    one, zero = Fraction(1), Fraction(0)
    classes = []
    for ct in plan.classes:
        T = tuple(tuple(Fraction(v) for v in row) + (zero,) for row in ct.T) + ((zero, zero, one),)
        pl = tuple(tuple(int(v) for v in row) + (0,) for row in ct.pi_linear) + ((0, 0, 1),)
        classes.append(ClassTransform(kernel=ct.kernel, T=T, t=tuple(ct.t) + (zero,), pi_linear=pl,
                                      pi_offset=tuple(ct.pi_offset) + (0,)))
    kernels = []
    for k in plan.kernels:
        groups = tuple(FetchGroup(tuple(tuple(s) + (0,) for s in g.sites), tuple(g.span_axes), _lift_poly(g.g),
                                  tuple(_lift_poly(t) for t in g.t_nums)) for g in k.groups)
        kernels.append(PlanKernel(k.ref_class, groups))
    return EvaluationPlan(
        name=plan.name,
        lattice_name=plan.lattice_name,
        s=3,
        diag=tuple(plan.diag) + (1,),
        shifts=tuple(tuple(sh) + (0,) for sh in plan.shifts),
        scale=plan.scale,
        planes=tuple((tuple(n) + (0,), off) for n, off in plan.planes),
        r=plan.r,
        sigma=tuple(plan.sigma),
        classes=tuple(classes),
        kernels=tuple(kernels),
        options=plan.options,
        basis_nonnegative=plan.basis_nonnegative,
        pou_on_sublattice=plan.pou_on_sublattice,
        reflective_axes=tuple(plan.reflective_axes) + (True,),
        octant_fold=plan.octant_fold,
    )


def lift_cosets(cos: CosetDecomposition) -> CosetDecomposition:
    L = cos.parent.L
    lat = IntegerLattice([list(row) + [0] for row in L] + [[0, 0, 1]], name=f"{cos.parent.name}x1")
    return CosetDecomposition(lat, tuple(cos.diag) + (1,), [tuple(sh) + (0,) for sh in cos.shifts])


def lift_grid(grid):
    """The grid as (n0, n1, 1) views over the caller's storage."""
    from .runtime import CoefficientGrid

    key = (id(grid), tuple(a.data_ptr() for a in grid.arrays))
    cached = getattr(grid, "_lifted", None)
    if cached is not None and cached[0] == key:
        return cached[1]
    g3 = CoefficientGrid(lift_cosets(grid.cosets), [a.unsqueeze(-1) for a in grid.arrays],
                         [tuple(o) + (0,) for o in grid.origins], grid.boundary, device=grid.device, dtype=grid.dtype)
    grid._lifted = (key, g3)
    return g3


def lift_points(pts):
    """(n, 2) points -> (n, 3) with third coordinate 0 (numpy -> float64 numpy, tensor ->
    tensor on the same device, same dtype)."""
    if isinstance(pts, torch.Tensor):
        return torch.cat([pts, torch.zeros((pts.shape[0], 1), dtype=pts.dtype, device=pts.device)], 1).contiguous()
    a = np.asarray(pts, dtype=np.float64)
    if a.ndim != 2 or a.shape[1] != 2:
        raise ValueError("points must have shape (n, 2)")
    return np.concatenate([a, np.zeros((a.shape[0], 1))], 1)
