"""CPU ORACLE (test infrastructure only) — numpy restatement of the reference batch path.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s cpu-baseline / `--impl reference`
leg may import this module, and only as the checker.  The product path never calls it.

What it restates (reference = splineplan 0.1.0, /root/reference/pkg/src/splineplan):

* `CoefficientGrid` storage, `_gather` boundary policies and `_mirror_index_array`
  (runtime.py:38-78, :151-168, :199-204);
* `fetch_nearest_batch` / `fetch_linear_batch` (runtime.py:170-188);
* `_poly_batch` monomial sums (runtime.py:345-360);
* `_eval_batch` — Algorithm 1 specialised per class (runtime.py:363-408), including the
  sigma-sentinel error (runtime.py:379-381) and the 0.5 texel round trip (:404-405);
* the per-coset (class id, kk) classification of runtime.py:371-379 as `classify_batch`.

It is the same sequence of float64 numpy operations as the reference, so it is
bit-identical to it on the committed golden vectors (tests/test_oracle_golden.py pins
that).  The third-party arithmetic is numpy (reference pins only numpy>=1.24,
pyproject.toml:11; fixtures were generated with numpy 2.3.5).
"""

from __future__ import annotations

import math
from itertools import product
from typing import Sequence

import numpy as np

BOUNDARIES = ("zero", "clamp", "mirror")


class OracleError(ValueError):
    """Stands in for the reference's RuntimeError_ (runtime.py:31-32)."""


class NumpyGrid:
    """Per-coset float64 C-order arrays + origins + boundary (runtime.py:38-63)."""

    def __init__(self, diag, shifts, arrays, origins, boundary="zero"):
        if boundary not in BOUNDARIES:
            raise OracleError(f"unknown boundary policy {boundary}")
        self.diag = tuple(int(d) for d in diag)
        self.shifts = tuple(tuple(int(v) for v in sh) for sh in shifts)
        self.arrays = [np.asarray(a, dtype=np.float64) for a in arrays]
        self.origins = [tuple(int(v) for v in o) for o in origins]
        self.boundary = boundary

    @staticmethod
    def zeros_extents(diag, shifts, lo, hi):
        """Origins/extents of CoefficientGrid.zeros (runtime.py:65-78)."""
        origins, extents = [], []
        for shift in shifts:
            zlo = [math.ceil((lo[i] - shift[i]) / d) for i, d in enumerate(diag)]
            zhi = [math.floor((hi[i] - shift[i]) / d) for i, d in enumerate(diag)]
            origins.append(tuple(zlo))
            extents.append(tuple(b - a + 1 for a, b in zip(zlo, zhi)))
        return origins, extents

    def _gather(self, coset: int, idx: np.ndarray) -> np.ndarray:
        """runtime.py:151-168."""
        arr = self.arrays[coset]
        n = idx.shape[0]
        if self.boundary == "zero":
            valid = np.ones(n, dtype=bool)
            for i, size in enumerate(arr.shape):
                valid &= (idx[:, i] >= 0) & (idx[:, i] < size)
            clipped = np.clip(idx, 0, np.array(arr.shape) - 1)
            vals = arr[tuple(clipped[:, i] for i in range(arr.ndim))]
            return np.where(valid, vals, 0.0)
        if self.boundary == "clamp":
            clipped = np.clip(idx, 0, np.array(arr.shape) - 1)
            return arr[tuple(clipped[:, i] for i in range(arr.ndim))]
        cols = [mirror_index_array(idx[:, i], size) for i, size in enumerate(arr.shape)]
        return arr[tuple(cols)]

    def fetch_nearest_batch(self, coset: int, z: np.ndarray) -> np.ndarray:
        """runtime.py:170-172 (rint = round half to even)."""
        idx = np.rint(z).astype(np.int64) - np.array(self.origins[coset])
        return self._gather(coset, idx)

    def fetch_linear_batch(self, coset: int, u: np.ndarray) -> np.ndarray:
        """runtime.py:174-188 with offset_half=False (the batch path pre-applies it)."""
        base = np.floor(u)
        frac = u - base
        base = base.astype(np.int64) - np.array(self.origins[coset])
        s = u.shape[1]
        total = np.zeros(u.shape[0])
        for corner in product((0, 1), repeat=s):
            w = np.ones(u.shape[0])
            for i, c in enumerate(corner):
                w = w * (frac[:, i] if c else 1.0 - frac[:, i])
            total += w * self._gather(coset, base + np.array(corner))
        return total


def mirror_index_array(v: np.ndarray, n: int) -> np.ndarray:
    """runtime.py:199-204 (period 2n-2)."""
    if n == 1:
        return np.zeros_like(v)
    period = 2 * n - 2
    v = np.abs(v) % period
    return np.where(v >= n, period - v, v)


class PlanTables:
    """Float tables of runtime.py:256-272 plus per-poly (exps, coeffs) of :345-353."""

    def __init__(self, plan):
        self.plan = plan
        s = plan.s
        self.normals = np.array([[float(v) for v in n] for n, _ in plan.planes]).reshape(plan.Q, s)
        self.offsets = np.array([float(o) for _, o in plan.planes])
        self.sigma = np.array(plan.sigma, dtype=np.int64)
        self.T = [np.array([[float(v) for v in row] for row in c.T]) for c in plan.classes]
        self.t = [np.array([float(v) for v in c.t]) for c in plan.classes]
        self.piA = [np.array([[int(v) for v in row] for row in c.pi_linear]) for c in plan.classes]
        self.pib = [np.array([int(v) for v in c.pi_offset]) for c in plan.classes]
        self._poly = {}

    def poly_arrays(self, poly):
        key = id(poly)
        hit = self._poly.get(key)
        if hit is None:
            exps = np.array(sorted(poly.terms), dtype=np.int64).reshape(len(poly.terms), poly.dim)
            coeffs = np.array([float(poly.terms[tuple(e)]) for e in exps])
            hit = (exps, coeffs)
            self._poly[key] = hit
        return hit


def poly_batch(poly, y: np.ndarray, tabs: PlanTables) -> np.ndarray:
    """runtime.py:356-360 — monomial sum, not Horner."""
    if not poly.terms:
        return np.zeros(y.shape[0])
    exps, coeffs = tabs.poly_arrays(poly)
    return np.power(y[:, None, :], exps[None, :, :]).prod(axis=2) @ coeffs


def _coset_frame(plan, pts, coset, tabs):
    """runtime.py:371-381: coset shift, rho, plane code, sigma."""
    diag = np.array(plan.diag, dtype=np.float64)
    xl = pts - np.array(plan.shifts[coset], dtype=np.float64)
    kk = np.floor(xl / diag) * diag
    xp = xl - kk
    n = pts.shape[0]
    if plan.Q:
        bits = (xp @ tabs.normals.T) >= tabs.offsets
        q = bits @ (1 << np.arange(plan.Q, dtype=np.int64))
    else:
        q = np.zeros(n, dtype=np.int64)
    cls = tabs.sigma[q % plan.r]
    return kk, xp, cls


def classify_batch(plan, pts: np.ndarray, tabs: PlanTables | None = None):
    """(n, M) class ids (-1 = sentinel) and (n, M, s) coset cells kk/d (runtime.py:371-379)."""
    tabs = tabs or PlanTables(plan)
    pts = np.asarray(pts, dtype=np.float64)
    diag = np.array(plan.diag, dtype=np.float64)
    classes = np.zeros((pts.shape[0], plan.M), dtype=np.int64)
    cells = np.zeros((pts.shape[0], plan.M, plan.s), dtype=np.int64)
    with np.errstate(invalid="ignore"):
        for k in range(plan.M):
            kk, _, cls = _coset_frame(plan, pts, k, tabs)
            classes[:, k] = cls
            cells[:, k, :] = (kk / diag).astype(np.int64)
    return classes, cells


def eval_batch(plan, grid: NumpyGrid, pts: np.ndarray, tabs: PlanTables | None = None) -> np.ndarray:
    """runtime.py:363-408, operation for operation."""
    if tuple(grid.diag) != tuple(plan.diag) or tuple(grid.shifts) != tuple(plan.shifts):
        raise OracleError("grid decomposition does not match the plan header")  # runtime.py:250-254
    tabs = tabs or PlanTables(plan)
    pts = np.asarray(pts, dtype=np.float64)
    n = pts.shape[0]
    out = np.zeros(n)
    diag = np.array(plan.diag, dtype=np.float64)
    offset = plan.options.texel_offset_half
    with np.errstate(divide="ignore", invalid="ignore"):
        for coset in range(plan.M):
            kk, xp, cls = _coset_frame(plan, pts, coset, tabs)
            if np.any(cls == -1):
                raise OracleError("sigma sentinel hit in batch evaluation")
            for c in np.unique(cls):
                sel = np.nonzero(cls == c)[0]
                ct = plan.classes[int(c)]
                y = xp[sel] @ tabs.T[c].T - tabs.t[c]
                kernel = plan.kernels[ct.kernel]
                A = tabs.piA[c]
                bvec = tabs.pib[c]
                acc = np.zeros(sel.size)
                for group in kernel.groups:
                    g = poly_batch(group.g, y, tabs)
                    mapped = [A @ np.array(site) + bvec for site in group.sites]
                    if not group.span_axes:
                        z = (mapped[0] + kk[sel]) / diag
                        acc += g * grid.fetch_nearest_batch(coset, z)
                    else:
                        base = (mapped[0] + kk[sel]) / diag
                        u = base.copy()
                        for j in range(len(group.span_axes)):
                            tnum = poly_batch(group.t_nums[j], y, tabs)
                            t = np.where(g == 0.0, 0.5, tnum / g)
                            corner = (mapped[1 << j] + kk[sel]) / diag
                            u = u + t[:, None] * (corner - base)
                        if offset:
                            u = (u + 0.5) - 0.5
                        acc += g * grid.fetch_linear_batch(coset, u)
                out[sel] += acc
    return out


def eval_batch_chunked(plan, grid: NumpyGrid, pts: np.ndarray, chunk: int = 1 << 15, tabs=None) -> np.ndarray:
    """Chunking is mandatory at scale; results are unchanged."""
    tabs = tabs or PlanTables(plan)
    pts = np.asarray(pts, dtype=np.float64)
    out = np.empty(pts.shape[0])
    for i in range(0, pts.shape[0], chunk):
        out[i : i + chunk] = eval_batch(plan, grid, pts[i : i + chunk], tabs)
    return out
