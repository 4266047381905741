"""Plans the REFERENCE compiles with non-default PlanOptions (build container only).

    python tests/golden/make_variant_golden.py

For small catalog splines: the reference's compile_plan (plancompile.py:339-380) over its own
analysis of the shipped PP document, for several option sets; the sha256 checksums of the
serialized plans go to tests/golden/variants.json (tests/test_variants.py derives the same
plans natively from the default catalog plan).
"""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "tools"))
from refshim import import_reference  # noqa: E402

LAT = {"zp": "CC2", "tp2": "CC2", "cc_trilinear": "CC3", "bcc_linear_rd": "BCC", "fcc_cubic": "FCC",
       "bcc_quintic_rd": "BCC"}
OPTS = [dict(grouped=False), dict(ordered=False), dict(grouped=False, ordered=False), dict(texel_offset_half=False),
        dict(predicated=False)]


def main():
    import_reference()
    from splineplan.analysis import enumerate_subregions, search_symmetry
    from splineplan.lattice import decompose_cartesian, named_lattice
    from splineplan.plancompile import PlanOptions, compile_plan, serialize_plan
    from splineplan.spline import SplineOnLattice, import_pp_spline

    out = {}
    for name, latname in LAT.items():
        sp = import_pp_spline(open(os.path.join(ROOT, "paper_2102_08514_b200", "pp", f"{name}.spp")).read(),
                              validate=False)
        lat = named_lattice(latname)
        sol = SplineOnLattice(sp, lat, decompose_cartesian(lat))
        roe = enumerate_subregions(sol)
        sym = search_symmetry(roe)
        for o in OPTS:
            plan = compile_plan(sol, roe, sym, options=PlanOptions(**o))
            key = name + ":" + ",".join(f"{k}={v}" for k, v in sorted(o.items()))
            out[key] = json.loads(serialize_plan(plan))["checksum"]
            print(key, out[key][:16], flush=True)
    with open(os.path.join(HERE, "variants.json"), "w") as fh:
        json.dump(out, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
