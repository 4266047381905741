"""Prefilter fixtures made with the REFERENCE's own primitives (build container only).

    python tests/golden/make_prefilter_golden.py

The reference ships the quasi-interpolation taps (`corpus.prefilter_taps`,
corpus.py:71-111) but no code that applies them (the convergence harness, SPEC.md:508-516,
is not shipped).  The application is the discrete lattice correlation

    out[site] = sum_o tap[o] * in[site + o]           (site, o on the lattice)

with `in` read through the reference's policy-aware `CoefficientGrid.site_value`
(runtime.py:94-97 -> _read_scalar :109-123).  This script evaluates exactly that, one site
at a time in pure Python over small seeded grids, with the reference's taps for
bcc_quintic_rd and the identity, plus asymmetric synthetic stencils that pin the sign
convention.  Output: tests/golden/prefilter/<case>.npz.
"""
import os
import sys

import numpy as np

GOLD = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(GOLD))
OUT = os.path.join(GOLD, "prefilter")
sys.path.insert(0, os.path.join(ROOT, "tools"))
from refshim import import_reference  # noqa: E402


def cases():
    from splineplan import corpus

    q = corpus.prefilter_taps("bcc_quintic_rd")
    ident = corpus.prefilter_taps("cc_trilinear")
    yield "bcc_quintic", "BCC", 9, {k: float(v) for k, v in q.items()}
    yield "identity_cc", "CC3", 6, {k: float(v) for k, v in ident.items()}
    yield "shift_cc", "CC3", 6, {(1, 0, 0): 1.0, (0, -2, 1): 0.5}
    yield "asym_fcc", "FCC", 7, {(0, 0, 0): 1.0, (1, 1, 0): 0.5, (-1, 0, 1): -0.25, (2, 0, 0): 0.125, (0, -1, -1): 2.0}
    yield "asym_bcc", "BCC", 7, {(1, 1, 1): 0.75, (-1, 1, -1): -1.5, (2, 0, 0): 0.25, (0, 0, -2): 1.0}


def main():
    import_reference()
    from splineplan.lattice import CoefficientIndex, decompose_cartesian, named_lattice
    from splineplan.runtime import CoefficientGrid

    os.makedirs(OUT, exist_ok=True)
    rng = np.random.default_rng(2102_08514 + 5)
    for name, lat_name, hi, taps in cases():
        cos = decompose_cartesian(named_lattice(lat_name))
        base = CoefficientGrid.zeros(cos, [0, 0, 0], [hi, hi, hi], "zero")
        arrays = [rng.random(a.shape, dtype=np.float32).astype(np.float64) for a in base.arrays]
        offs = sorted(taps)
        payload = dict(lattice=np.array(lat_name), offsets=np.array(offs, dtype=np.int64),
                       taps=np.array([taps[o] for o in offs]), origins=np.array(base.origins, dtype=np.int64))
        for k, a in enumerate(arrays):
            payload[f"in{k}"] = a
        for boundary in ("zero", "clamp", "mirror"):
            grid = CoefficientGrid(cos, arrays, base.origins, boundary)
            for k, a in enumerate(arrays):
                out = np.zeros_like(a)
                for z in np.ndindex(*a.shape):
                    cell = tuple(int(v) + o for v, o in zip(z, base.origins[k]))
                    site = cos.site_of(CoefficientIndex(k, cell))
                    acc = 0.0
                    for o in offs:
                        acc += taps[o] * grid.site_value([s + d for s, d in zip(site, o)])
                    out[z] = acc
                payload[f"out_{boundary}{k}"] = out
        np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **payload)
        print(name, [a.shape for a in arrays])


if __name__ == "__main__":
    main()
