"""Quasi-interpolation prefilter on coset grids — the step before
reconstruction in the paper's convergence study (§5.2).

`prefilter_taps(name)` gives the reference's taps (corpus.py:71-111: a {lattice offset:
rational} map, identity when the spline needs none).  `apply_prefilter(grid, taps)`
returns a new `CoefficientGrid` holding the lattice correlation

    out[site] = sum_o tap[o] * in[site + o]        (offsets in sorted order)

with the input read through the grid's boundary policy (runtime.py:109-123).  The work
runs in libsplinerecon.so (`sp_prefilter`): the offsets are resolved once on the host
into per-output-coset (source coset, cell offset, weight) taps, the device kernel is a
streaming stencil (one read of each input coset, one write of each output coset from
HBM).  float64 grids reproduce the reference's per-site loop bit for bit
(tests/test_prefilter.py); float32 grids compute in float32.
"""

from __future__ import annotations

import ctypes
from fractions import Fraction
from typing import Mapping

import numpy as np
import torch

from . import _native
from .corpus import prefilter_taps  # noqa: F401  (re-export: corpus.prefilter_taps)
from .runtime import CoefficientGrid, RuntimeError_


def stencil_taps(cosets, taps: Mapping) -> list:
    """Per output coset k: [(source coset, (dz0, dz1, dz2), weight)] in sorted-offset order.
    site = D z + l_k; site + o = D (z + dz) + l_k' with dz = (l_k + o - l_k') / D."""
    diag = [int(d) for d in cosets.diag]
    shifts = [tuple(int(v) for v in s) for s in cosets.shifts]
    table = []
    for lk in shifts:
        rows = []
        for o in sorted(tuple(int(v) for v in off) for off in taps):
            w = taps[o] if o in taps else taps[tuple(o)]
            p = [a + b for a, b in zip(lk, o)]
            for kk, l2 in enumerate(shifts):
                if all((x - l) % d == 0 for x, l, d in zip(p, l2, diag)):
                    rows.append((kk, tuple((x - l) // d for x, l, d in zip(p, l2, diag)), float(Fraction(w))))
                    break
            else:
                raise RuntimeError_(f"prefilter offset {o} is not a lattice vector")
        table.append(rows)
    return table


def apply_prefilter(grid: CoefficientGrid, taps: Mapping, *, out: CoefficientGrid | None = None,
                    stream: torch.cuda.Stream | None = None) -> CoefficientGrid:
    """Prefiltered copy of `grid` (same cosets, origins, extents, dtype, boundary)."""
    s = grid.cosets.parent.s
    if s != 3:
        raise NotImplementedError("prefilter: 3-D grids only (every BASELINE config is 3-D)")
    if any(len(o) != s for o in taps):
        raise RuntimeError_("prefilter offsets must have the grid's dimension")
    table = stencil_taps(grid.cosets, taps)
    if max(len(r) for r in table) > _native.SP_MAX_STENCIL:
        raise RuntimeError_(f"at most {_native.SP_MAX_STENCIL} taps per coset")
    if out is None:
        out = CoefficientGrid(grid.cosets, [torch.empty_like(a) for a in grid.arrays], grid.origins, grid.boundary,
                              device=grid.device, dtype=grid.dtype)
    elif [tuple(a.shape) for a in out.arrays] != [tuple(a.shape) for a in grid.arrays] or out.dtype != grid.dtype:
        raise RuntimeError_("output grid must match the input grid's extents and dtype")
    if any(a.data_ptr() == b.data_ptr() for a in out.arrays for b in grid.arrays):
        raise RuntimeError_("prefilter output must not alias its input")
    src = np.array([t[0] for r in table for t in r], dtype=np.int32)
    dz = np.array([t[1] for r in table for t in r], dtype=np.int32).reshape(-1, 3)
    w = np.array([t[2] for r in table for t in r], dtype=np.float64)
    d = _native.StencilDesc()
    d.M = grid.cosets.M
    acc = 0
    for k, r in enumerate(table):
        d.tap_start[k] = acc
        acc += len(r)
    d.tap_start[len(table)] = acc
    src = np.ascontiguousarray(src)
    dz = np.ascontiguousarray(dz)
    w = np.ascontiguousarray(w)
    d.src_coset = src.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))
    d.dz = dz.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))
    d.weight = w.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
    outs = (ctypes.c_void_p * _native.SP_MAX_COSETS)(*([a.data_ptr() for a in out.arrays] +
                                                      [0] * (_native.SP_MAX_COSETS - len(out.arrays))))
    st = stream if stream is not None else torch.cuda.current_stream(grid.device)
    gdesc = grid.descriptor()
    _native.check(_native.lib().sp_prefilter(ctypes.byref(gdesc), ctypes.byref(d), outs, st.cuda_stream))
    return out
