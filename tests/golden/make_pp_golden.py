"""Reference values for the PP-form API (build container only).

    python tests/golden/make_pp_golden.py

For the shipped PP documents (paper_2102_08514_b200/pp/*.spp): the REFERENCE's
import_pp_spline (spline.py:667-713) + eval_exact (spline.py:391-395) at seeded rational
points, and its SplineOnLattice.contributing_sites (spline.py:599-610) — frozen as strings in
tests/golden/pp_values.json for tests/test_pp.py.
"""
import json
import os
import random
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "tools"))
from refshim import import_reference  # noqa: E402

PP = os.path.join(ROOT, "paper_2102_08514_b200", "pp")
LAT = {"tp2": "CC2", "zp": "CC2", "qc_tensor": "QC", "cc_trilinear": "CC3", "bcc_linear_rd": "BCC",
       "bcc_quintic_rd": "BCC", "fcc_cubic": "FCC", "cc_tricubic": "CC3", "cc_zp3": "CC3", "bcc_quartic": "BCC",
       "fcc_voronoi1": "FCC", "bcc_voronoi1": "BCC"}


def main():
    import_reference()
    from fractions import Fraction

    from splineplan.exactmath import rat_to_str
    from splineplan.lattice import decompose_cartesian, named_lattice
    from splineplan.spline import SplineOnLattice, import_pp_spline

    out = {}
    for f in sorted(os.listdir(PP)):
        name = f[: -len(".spp")]
        sp = import_pp_spline(open(os.path.join(PP, f)).read(), validate=False)
        lat = named_lattice(LAT[name])
        sol = SplineOnLattice(sp, lat, decompose_cartesian(lat))
        rng = random.Random(sum(map(ord, name)))
        lo, hi = sp.support.bbox()
        pts = [tuple(Fraction(rng.randint(int(l * 8) - 4, int(h * 8) + 4), 8) for l, h in zip(lo, hi)) for _ in range(24)]
        pts += [tuple(Fraction(rng.randint(-300, 300), 97) for _ in range(sp.s)) for _ in range(8)]
        vals = [rat_to_str(sp.eval_exact(p)) for p in pts]
        sites = [sol.contributing_sites(p) for p in pts[-4:]]
        out[name] = {"pieces": len(sp.pieces), "points": [[rat_to_str(v) for v in p] for p in pts], "values": vals,
                     "sites": [[list(s) for s in ss] for ss in sites]}
        print(name, len(sp.pieces), flush=True)
    with open(os.path.join(HERE, "pp_values.json"), "w") as fh:
        json.dump(out, fh, indent=0, sort_keys=True)


if __name__ == "__main__":
    main()
