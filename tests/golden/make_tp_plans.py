"""Freeze reference-compiled tensor-product B-spline plans (E3 x (n+1) on CC3) as golden
fixtures for the native plan producer (paper_2102_08514_b200/tpplan.py).

Runs only in the build container (imports /root/reference through tools/refshim.py):
PP extraction (spline.py:481-531), sub-region analysis and symmetry search
(analysis.py:113-399) and compile_plan (plancompile.py:328-380) with default PlanOptions,
then serialize_plan — exactly the path tools/gen_plans.py takes for cc_tricubic.

usage: python tests/golden/make_tp_plans.py 2 4 [...]   -> tests/golden/tp_plans/cc_tp<n>.plan.json
"""
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", "..", "tools"))
from refshim import import_reference  # noqa: E402

OUT = os.path.join(HERE, "tp_plans")
E3 = [(1, 0, 0), (0, 1, 0), (0, 0, 1)]


def build(n: int) -> None:
    import_reference()
    from splineplan.analysis import enumerate_subregions, search_symmetry
    from splineplan.lattice import decompose_cartesian, named_lattice
    from splineplan.plancompile import compile_plan, serialize_plan
    from splineplan.spline import DirectionMatrix, SplineOnLattice, extract_pp_form

    t0 = time.time()
    name = f"cc_tp{n}"
    sp = extract_pp_form(DirectionMatrix(E3 * (n + 1)), name=name)
    lat = named_lattice("CC3")
    sol = SplineOnLattice(sp, lat, decompose_cartesian(lat))
    roe = enumerate_subregions(sol)
    sym = search_symmetry(roe)
    plan = compile_plan(sol, roe, sym)
    os.makedirs(OUT, exist_ok=True)
    with open(os.path.join(OUT, f"{name}.plan.json"), "w") as fh:
        fh.write(serialize_plan(plan))
    print(f"[{name}] {len(sp.pieces)} pieces, K={plan.K}, groups={len(plan.kernels[0].groups)} "
          f"in {time.time() - t0:.1f}s", flush=True)


if __name__ == "__main__":
    for a in sys.argv[1:]:
        build(int(a))
