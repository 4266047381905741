"""Reference plans for box splines outside the catalog (build container only).

    python tests/golden/make_boxplan_golden.py

Runs the REFERENCE pipeline end to end — DirectionMatrix -> extract_pp_form (spline.py:481-531)
-> SplineOnLattice -> enumerate_subregions / search_symmetry (analysis.py:113-399) ->
compile_plan (plancompile.py:339-380) -> serialize_plan — for direction sets the shipped
catalog does not hold, and freezes the documents (plus the PP documents, format_pp_spline)
under tests/golden/boxplan/.  tests/test_boxplan.py checks that boxplan.box_spline_plan
produces the same plans and documents without the reference.
"""
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "tools"))
from refshim import import_reference  # noqa: E402

OUT = os.path.join(HERE, "boxplan")

E3 = [(1, 0, 0), (0, 1, 0), (0, 0, 1)]
CASES = {
    # name: (direction columns, lattice)
    "cc2_courant": ([(1, 0), (0, 1), (1, 1)], "CC2"),
    "cc2_biquadratic": ([(1, 0), (0, 1)] * 3, "CC2"),
    "qc_zp": ([(1, 0), (0, 1), (1, 1), (-1, 1)], "QC"),
    "cc2_hex3": ([(1, 0), (0, 1), (1, 1)] * 2, "CC2"),
    "cc3_e3_d1": (E3 + [(1, 1, 1)], "CC3"),
    "cc3_e3_d2": (E3 + [(1, 1, 1), (1, -1, 1)], "CC3"),
}
# E3 x 2 on FCC is not a partition of unity: the reference raises SplineError in
# enumerate_subregions (analysis.py:124); tests/test_boxplan.py expects the same refusal.


def main(names):
    import_reference()
    from splineplan.analysis import enumerate_subregions, search_symmetry
    from splineplan.lattice import decompose_cartesian, named_lattice
    from splineplan.plancompile import compile_plan, serialize_plan
    from splineplan.spline import DirectionMatrix, SplineOnLattice, extract_pp_form, format_pp_spline

    os.makedirs(OUT, exist_ok=True)
    for name in names or sorted(CASES):
        cols, latname = CASES[name]
        t0 = time.time()
        sp = extract_pp_form(DirectionMatrix(cols), name=name)
        lat = named_lattice(latname)
        sol = SplineOnLattice(sp, lat, decompose_cartesian(lat))
        roe = enumerate_subregions(sol)
        sym = search_symmetry(roe)
        plan = compile_plan(sol, roe, sym)
        with open(os.path.join(OUT, f"{name}.spp"), "w") as fh:
            fh.write(format_pp_spline(sp))
        with open(os.path.join(OUT, f"{name}.plan.json"), "w") as fh:
            fh.write(serialize_plan(plan))
        print(f"{name}: pieces={len(sp.pieces)} N={roe.N} K={sym.K} ({time.time() - t0:.1f}s)", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:])
