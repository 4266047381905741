"""Freeze the PP forms (the reference's `.spp` import/cache documents) of the catalog splines
(build container only; needs /root/reference).

    python tools/gen_pp.py [name ...]

Each document is the reference's own `extract_pp_form` (spline.py:481-531) rendered by
`format_pp_spline` (spline.py:645-664) — exactly what the reference's `build_spline` caches
(corpus.py:124-138) — written to paper_2102_08514_b200/pp/<name>.spp, where the drop-in's
`corpus.build_spline` / `build_pair` load them.  The Voronoi documents come from
tools/voronoi_pp.py.
"""
import os
import shutil
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from refshim import import_reference  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "paper_2102_08514_b200", "pp")
E3 = [(1, 0, 0), (0, 1, 0), (0, 0, 1)]
DIAG = [(1, 1, 1), (-1, 1, 1), (1, -1, 1), (1, 1, -1)]
EXTRA = {"cc_tricubic": E3 * 4, "cc_zp3": E3 + DIAG, "bcc_quartic": DIAG + [(2, 0, 0), (0, 2, 0), (0, 0, 2)]}


def main(names):
    import_reference()
    from splineplan import corpus
    from splineplan.spline import DirectionMatrix, extract_pp_form, format_pp_spline

    os.makedirs(OUT, exist_ok=True)
    names = names or list(corpus.DIRECTION_SETS) + list(EXTRA)
    for name in names:
        if name == "d4_order4":
            continue  # 4-D: no compiled plan, out of scope
        t0 = time.time()
        cache = os.path.join(os.environ["SPLINEPLAN_CACHE"], f"{name}.spp")
        if os.path.exists(cache):
            shutil.copy(cache, os.path.join(OUT, f"{name}.spp"))
        else:
            cols = corpus.DIRECTION_SETS[name][0] if name in corpus.DIRECTION_SETS else EXTRA[name]
            sp = extract_pp_form(DirectionMatrix(cols), name=name)
            with open(os.path.join(OUT, f"{name}.spp"), "w") as fh:
                fh.write(format_pp_spline(sp))
        print(f"[{name}] {time.time() - t0:.1f}s", flush=True)
    for v in ("fcc_voronoi1", "bcc_voronoi1"):
        shutil.copy(os.path.join(ROOT, "tests", "golden", "voronoi", f"{v}.spp"), os.path.join(OUT, f"{v}.spp"))


if __name__ == "__main__":
    main(sys.argv[1:])
