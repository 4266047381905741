"""CPU ORACLE (test infrastructure only) — quasi-interpolation prefilter on coset grids.

Only tests/ (and bench.py's CPU leg) may import this module, as the checker.

The reference ships the taps (`corpus.prefilter_taps`, corpus.py:71-111) and the
policy-aware site read (`CoefficientGrid.site_value` -> `_read_scalar`, runtime.py:94-123)
but no code that applies the taps (the convergence harness, is not
shipped).  The application restated here is the discrete lattice correlation

    out[site] = sum over offsets o (sorted) of tap[o] * in[site + o]

evaluated per output coset k over its whole array: site = D (z + origin_k) + l_k, the
source site + o lies on coset k' with cell z + origin_k + dz, dz = (l_k + o - l_k') / D.
The sum runs in sorted-offset order with separate multiply and add, i.e. exactly the
float64 operations of the per-site loop in tests/golden/make_prefilter_golden.py, which
ran it through the reference's own `site_value` — so this restatement is bit-identical to
those fixtures (tests/test_prefilter.py pins it).
"""

from __future__ import annotations

import numpy as np

from .plan_numpy import NumpyGrid


def stencil_table(diag, shifts, offsets, taps):
    """Per output coset: [(source coset, dz (3,), tap)] in sorted-offset order."""
    diag = [int(d) for d in diag]
    shifts = [tuple(int(v) for v in s) for s in shifts]
    order = sorted(range(len(offsets)), key=lambda i: tuple(int(v) for v in offsets[i]))
    table = []
    for lk in shifts:
        rows = []
        for i in order:
            o = [int(v) for v in offsets[i]]
            p = [a + b for a, b in zip(lk, o)]
            for kk, l2 in enumerate(shifts):
                if all((x - l) % d == 0 for x, l, d in zip(p, l2, diag)):
                    rows.append((kk, tuple((x - l) // d for x, l, d in zip(p, l2, diag)), float(taps[i])))
                    break
            else:
                raise ValueError(f"offset {o} does not map coset shift {lk} onto the lattice")
        table.append(rows)
    return table


def apply_prefilter(grid: NumpyGrid, offsets, taps) -> list:
    """Prefiltered coset arrays (float64), same shapes / origins / policy as `grid`."""
    table = stencil_table(grid.diag, grid.shifts, offsets, taps)
    outs = []
    for k, arr in enumerate(grid.arrays):
        z = np.stack(np.meshgrid(*[np.arange(n) for n in arr.shape], indexing="ij"), -1).reshape(-1, arr.ndim)
        cells = z + np.array(grid.origins[k])
        acc = np.zeros(z.shape[0])
        for kk, dz, w in table[k]:
            idx = cells + np.array(dz) - np.array(grid.origins[kk])
            acc = acc + w * grid._gather(kk, idx)
        outs.append(acc.reshape(arr.shape))
    return outs
