"""Flatten an EvaluationPlan into the C-ABI descriptor arrays (include/splinerecon.h).

Floats are `float(Fraction)` exactly as the reference lowers them (runtime.py:256-272,
:345-353); the same arrays feed both `sp_plan_create` (via ctypes) and the build-time
code generator, whose kernel registry is matched on `canonical_words` — the identical
word sequence splinerecon.cu:canonical_words() builds from the descriptor.
"""

from __future__ import annotations

import struct
from dataclasses import dataclass

import numpy as np

from .plan import EvaluationPlan

SP_MAX_DIM = 3


@dataclass
class PackedPlan:
    s: int
    M: int
    diag: list
    shifts: list
    Q: int
    normals: np.ndarray
    offsets: np.ndarray
    r: int
    sigma: np.ndarray
    N: int
    cls_kernel: np.ndarray
    cls_T: np.ndarray
    cls_t: np.ndarray
    cls_piA: np.ndarray
    cls_pib: np.ndarray
    K: int
    kernel_group_start: np.ndarray
    n_groups: int
    group_span: np.ndarray
    group_nspan: np.ndarray
    group_site_start: np.ndarray
    sites: np.ndarray
    group_poly_start: np.ndarray
    n_polys: int
    poly_term_start: np.ndarray
    term_exps: np.ndarray
    term_coeffs: np.ndarray
    texel_offset_half: int


def pack_plan(plan: EvaluationPlan) -> PackedPlan:
    s = plan.s
    i32 = lambda v: np.ascontiguousarray(np.array(v, dtype=np.int32).ravel())  # noqa: E731
    f64 = lambda v: np.ascontiguousarray(np.array(v, dtype=np.float64).ravel())  # noqa: E731
    kgs = [0]
    spans, nspan, gss, sites, gps, pts_, exps, coeffs = [], [], [0], [], [0], [0], [], []
    n_polys = 0
    for kern in plan.kernels:
        for g in kern.groups:
            nspan.append(len(g.span_axes))
            spans.extend(list(g.span_axes) + [-1] * (SP_MAX_DIM - len(g.span_axes)))
            for site in g.sites:
                sites.extend(site)
            gss.append(gss[-1] + len(g.sites))
            for poly in (g.g,) + tuple(g.t_nums):
                for e in sorted(poly.terms):
                    exps.extend(e)
                    coeffs.append(float(poly.terms[e]))
                pts_.append(len(coeffs))
                n_polys += 1
            gps.append(n_polys)
        kgs.append(len(nspan))
    return PackedPlan(
        s=s,
        M=plan.M,
        diag=list(plan.diag),
        shifts=[list(sh) for sh in plan.shifts],
        Q=plan.Q,
        normals=i32([list(n) for n, _ in plan.planes]),
        offsets=f64([float(o) for _, o in plan.planes]),
        r=plan.r,
        sigma=i32(plan.sigma),
        N=plan.N,
        cls_kernel=i32([c.kernel for c in plan.classes]),
        cls_T=f64([[float(v) for v in row] for c in plan.classes for row in c.T]),
        cls_t=f64([float(v) for c in plan.classes for v in c.t]),
        cls_piA=i32([[int(v) for v in row] for c in plan.classes for row in c.pi_linear]),
        cls_pib=i32([int(v) for c in plan.classes for v in c.pi_offset]),
        K=plan.K,
        kernel_group_start=i32(kgs),
        n_groups=len(nspan),
        group_span=i32(spans),
        group_nspan=i32(nspan),
        group_site_start=i32(gss),
        sites=i32(sites),
        group_poly_start=i32(gps),
        n_polys=n_polys,
        poly_term_start=i32(pts_),
        term_exps=i32(exps),
        term_coeffs=f64(coeffs),
        texel_offset_half=int(plan.options.texel_offset_half),
    )


def _u64_of_double(v: float) -> int:
    return struct.unpack("<Q", struct.pack("<d", float(v)))[0]


def canonical_words(p: PackedPlan) -> list:
    """Mirror of splinerecon.cu canonical_words(): ints as two's-complement uint64,
    doubles by bit pattern, in a fixed field order."""
    w = []
    I = lambda v: w.append(int(v) & 0xFFFFFFFFFFFFFFFF)  # noqa: E731
    D = lambda v: w.append(_u64_of_double(v))  # noqa: E731
    s = p.s
    I(s)
    I(p.M)
    for i in range(s):
        I(p.diag[i])
    for k in range(p.M):
        for i in range(s):
            I(p.shifts[k][i])
    I(p.Q)
    for v in p.normals:
        I(v)
    for v in p.offsets:
        D(v)
    I(p.r)
    for v in p.sigma:
        I(v)
    I(p.N)
    for v in p.cls_kernel:
        I(v)
    for v in p.cls_T:
        D(v)
    for v in p.cls_t:
        D(v)
    for v in p.cls_piA:
        I(v)
    for v in p.cls_pib:
        I(v)
    I(p.K)
    for v in p.kernel_group_start:
        I(v)
    I(p.n_groups)
    for v in p.group_nspan:
        I(v)
    for v in p.group_span:
        I(v)
    for v in p.group_site_start:
        I(v)
    for v in p.sites:
        I(v)
    for v in p.group_poly_start:
        I(v)
    I(p.n_polys)
    for v in p.poly_term_start:
        I(v)
    for v in p.term_exps:
        I(v)
    for v in p.term_coeffs:
        D(v)
    return w
