"""Compile evaluation plans with the reference compiler and freeze them as JSON.

Runs only in the build container (needs /root/reference).  Output goes to
paper_2102_08514_b200/plans/<name>.plan.json in the reference's own wire format
(`serialize_plan`, plancompile.py:535-539), checksum included.

Corpus splines use `corpus.build_plan` (corpus.py:153-156).  The two BASELINE
splines that are not in the corpus are built through the public API exactly as
SURVEY.md §9 describes:  cc_tricubic = E3x4, cc_zp3 = E3 + 4 body diagonals.

usage: python tools/gen_plans.py NAME [NAME ...]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from refshim import import_reference  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2102_08514_b200", "plans")

E3 = [(1, 0, 0), (0, 1, 0), (0, 0, 1)]
DIAG = [(1, 1, 1), (-1, 1, 1), (1, -1, 1), (1, 1, -1)]
EXTRA = {
    "cc_tricubic": (E3 * 4, "CC3"),
    "cc_triquadratic": (E3 * 3, "CC3"),
    "cc_zp3": (E3 + DIAG, "CC3"),
    "bcc_quartic": (DIAG + [(2, 0, 0), (0, 2, 0), (0, 0, 2)], "BCC"),
}
# Voronoi splines: PP data built by tools/voronoi_pp.py from the reference's exact tools
# and imported through the reference's own import path (spline.py:667-713).
VORONOI = {"fcc_voronoi1": "FCC", "bcc_voronoi1": "BCC"}
SPP_DIR = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden", "voronoi")


def build(name: str, grouped: bool = True):
    import_reference()
    from splineplan import corpus
    from splineplan.analysis import enumerate_subregions, search_symmetry
    from splineplan.lattice import decompose_cartesian, named_lattice
    from splineplan.plancompile import compile_plan, serialize_plan
    from splineplan.spline import DirectionMatrix, SplineOnLattice, extract_pp_form, format_pp_spline

    t0 = time.time()
    if name in corpus.DIRECTION_SETS:
        plan = corpus.build_plan(name)
    elif name in VORONOI:
        from splineplan.plancompile import PlanOptions
        from splineplan.spline import import_pp_spline

        sp = import_pp_spline(open(os.path.join(SPP_DIR, f"{name}.spp")).read(), validate=True)
        print(f"[{name}] imported {len(sp.pieces)} pieces in {time.time()-t0:.1f}s", flush=True)
        lat = named_lattice(VORONOI[name])
        sol = SplineOnLattice(sp, lat, decompose_cartesian(lat))
        roe = enumerate_subregions(sol)
        print(f"[{name}] N={roe.N} Q={roe.Q} r={roe.r} ({time.time()-t0:.1f}s)", flush=True)
        sym = search_symmetry(roe)
        print(f"[{name}] K={sym.K} ({time.time()-t0:.1f}s)", flush=True)
        plan = compile_plan(sol, roe, sym, options=PlanOptions(grouped=grouped))
    else:
        cols, latname = EXTRA[name]
        cache = os.path.join(os.environ["SPLINEPLAN_CACHE"], f"{name}.spp")
        if os.path.exists(cache):
            from splineplan.spline import import_pp_spline
            sp = import_pp_spline(open(cache).read(), validate=False)
        else:
            sp = extract_pp_form(DirectionMatrix(cols), name=name)
            os.makedirs(os.path.dirname(cache), exist_ok=True)
            with open(cache, "w") as fh:
                fh.write(format_pp_spline(sp))
        print(f"[{name}] extracted {len(sp.pieces)} pieces in {time.time()-t0:.1f}s", flush=True)
        lat = named_lattice(latname)
        sol = SplineOnLattice(sp, lat, decompose_cartesian(lat))
        roe = enumerate_subregions(sol)
        print(f"[{name}] N={roe.N} Q={roe.Q} r={roe.r} ({time.time()-t0:.1f}s)", flush=True)
        sym = search_symmetry(roe)
        print(f"[{name}] K={sym.K} ({time.time()-t0:.1f}s)", flush=True)
        from splineplan.plancompile import PlanOptions

        plan = compile_plan(sol, roe, sym, options=PlanOptions(grouped=grouped))
    os.makedirs(OUT, exist_ok=True)
    out_name = name if grouped else f"{name}_ungrouped"
    with open(os.path.join(OUT, f"{out_name}.plan.json"), "w") as fh:
        fh.write(serialize_plan(plan))
    print(f"[{name}] done in {time.time()-t0:.1f}s  M={plan.M} N={plan.N} Q={plan.Q} r={plan.r} K={plan.K}", flush=True)


if __name__ == "__main__":
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    for n in args:
        build(n, grouped="--ungrouped" not in sys.argv)
