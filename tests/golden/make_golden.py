"""Generate the golden fixtures by running the REFERENCE itself (build container only).

    python tests/golden/make_golden.py [name ...]

For every plan in paper_2102_08514_b200/plans/ (compiled by tools/gen_plans.py with the
reference compiler) this writes tests/golden/<name>.npz holding:

* a seeded small coefficient grid built with the reference `CoefficientGrid.zeros`
  (runtime.py:65-78); values are float32-representable so the fp32 device grid is the
  same grid;
* seeded float32 query points: uniform points overlapping the domain edges, dyadic
  points on plane ties / coset-cell faces, and far out-of-domain points;
* `PlanInterpreter.eval_batch` outputs (runtime.py:244-248) for each boundary policy;
* per-coset class ids and cells from the reference's own batch tables (runtime.py:371-379);
* `PlanInterpreter.eval` (scalar, runtime.py:232-242) and `eval_bruteforce`
  (runtime.py:415-427) on a subsample, when the PP form is available.

The fixtures travel to the GPU box; /root/reference does not.
"""

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "tools"))
from refshim import import_reference  # noqa: E402

PLANS = os.path.join(ROOT, "paper_2102_08514_b200", "plans")

E3 = [(1, 0, 0), (0, 1, 0), (0, 0, 1)]
DIAG = [(1, 1, 1), (-1, 1, 1), (1, -1, 1), (1, 1, -1)]
EXTRA = {"cc_tricubic": E3 * 4, "cc_zp3": E3 + DIAG, "bcc_quartic": DIAG + E3 + E3}
VORONOI_LAT = {"fcc_voronoi1": "FCC", "bcc_voronoi1": "BCC"}
EXTRA_LAT = {"cc_tricubic": "CC3", "cc_zp3": "CC3", "bcc_quartic": "BCC"}

# grid hi per lattice (lo = 0): small enough for brute force, large enough for halos
HI = {"CC3": 11, "BCC": 13, "FCC": 13, "CC2": 11, "QC": 11}


def _sol(name, ref):
    name = name.replace("_ungrouped", "")
    from splineplan import corpus
    from splineplan.lattice import decompose_cartesian, named_lattice
    from splineplan.spline import SplineOnLattice, import_pp_spline

    if name in corpus.DIRECTION_SETS:
        return corpus.build_pair(name)
    if name in VORONOI_LAT:
        # PP data made by tools/voronoi_pp.py, imported through spline.py:667-713
        sp = import_pp_spline(open(os.path.join(HERE, "voronoi", f"{name}.spp")).read(), validate=False)
        lat = named_lattice(VORONOI_LAT[name])
        return SplineOnLattice(sp, lat, decompose_cartesian(lat))
    cache = os.path.join(os.environ["SPLINEPLAN_CACHE"], f"{name}.spp")
    if not os.path.exists(cache):
        return None
    sp = import_pp_spline(open(cache).read(), validate=False)
    lat = named_lattice(EXTRA_LAT[name])
    return SplineOnLattice(sp, lat, decompose_cartesian(lat))


def make(name: str, seed: int):
    ref = import_reference()
    from splineplan.lattice import decompose_cartesian, named_lattice
    from splineplan.plancompile import deserialize_plan
    from splineplan.runtime import CoefficientGrid, PlanInterpreter, eval_bruteforce, eval_bruteforce_exact

    t0 = time.time()
    text = open(os.path.join(PLANS, f"{name}.plan.json")).read()
    plan = deserialize_plan(text)
    s = plan.s
    lat = named_lattice(plan.lattice_name)
    cos = decompose_cartesian(lat)
    hi = HI[plan.lattice_name]
    rng = np.random.default_rng(seed)

    grids = {}
    base = CoefficientGrid.zeros(cos, [0] * s, [hi] * s, "zero")
    arrays32 = [rng.random(a.shape, dtype=np.float32) for a in base.arrays]
    for b in ("zero", "clamp", "mirror"):
        grids[b] = CoefficientGrid(cos, [a.astype(np.float64) for a in arrays32], base.origins, b)

    # query points (float32, upcast exactly to float64 as in the reference, runtime.py:248)
    n_uni = 4096
    uni = rng.uniform(-2.5, hi + 2.5, size=(n_uni, s)).astype(np.float32)
    dy = (np.round(rng.uniform(-1.0, hi + 1.0, size=(1024, s)) * 4) / 4).astype(np.float32)  # plane ties
    ints = np.round(rng.uniform(0, hi, size=(256, s))).astype(np.float32)  # cell corners
    far = rng.uniform(-40, hi + 40, size=(128, s)).astype(np.float32)  # far outside (policies)
    tiny = (rng.uniform(-1, 1, size=(128, s)) * np.float32(2.0) ** rng.integers(-30, 0, size=(128, s))).astype(
        np.float32
    )  # |x| << 1: exercises the x - shift rounding corner
    pts = np.concatenate([uni, dy, ints, far, tiny]).astype(np.float32)
    p64 = pts.astype(np.float64)

    interp = PlanInterpreter(plan)
    outs = {b: interp.eval_batch(grids[b], p64) for b in grids}

    # classification straight from the reference's tables and runtime.py:371-379 lines
    tabs = interp._batch_tables()
    diag = np.array(plan.diag, dtype=np.float64)
    classes = np.zeros((pts.shape[0], plan.M), dtype=np.int64)
    cells = np.zeros((pts.shape[0], plan.M, s), dtype=np.int64)
    for coset, shift in enumerate(plan.shifts):
        xl = p64 - np.array(shift, dtype=np.float64)
        kk = np.floor(xl / diag) * diag
        xp = xl - kk
        if plan.Q:
            bits = (xp @ tabs["normals"].T) >= tabs["offsets"]
            q = bits @ (1 << np.arange(plan.Q, dtype=np.int64))
        else:
            q = np.zeros(pts.shape[0], dtype=np.int64)
        classes[:, coset] = tabs["sigma"][q % plan.r]
        cells[:, coset] = (kk / diag).astype(np.int64)

    # scalar path + brute force on a subsample
    sub = np.arange(0, n_uni, max(1, n_uni // 48))[:48]
    scalar = np.array([interp.eval(grids["zero"], list(map(float, p64[i]))) for i in sub])
    brute = np.full(sub.shape, np.nan)
    exact = np.full(sub.shape, np.nan)
    sol = _sol(name, ref)
    if sol is not None:
        from fractions import Fraction

        brute = np.array(
            [eval_bruteforce(sol, grids["zero"], [Fraction(float(v)) for v in p64[i]]) for i in sub]
        )
        # exact rational convolution sum (runtime.py:430-439), rounded once to float64
        exact = np.array(
            [float(eval_bruteforce_exact(sol, grids["zero"], [Fraction(float(v)) for v in p64[i]])) for i in sub]
        )

    payload = dict(
        name=np.array(name),
        pts=pts,
        origins=np.array(base.origins, dtype=np.int64),
        n_cosets=np.array(plan.M),
        out_zero=outs["zero"],
        out_clamp=outs["clamp"],
        out_mirror=outs["mirror"],
        classes=classes,
        cells=cells,
        sub=sub,
        scalar=scalar,
        brute=brute,
        exact=exact,
        numpy_version=np.array(np.__version__),
    )
    for k, a in enumerate(arrays32):
        payload[f"coset{k}"] = a
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **payload)
    err = np.nanmax(np.abs(brute - outs["zero"][sub])) if sol is not None else float("nan")
    errx = np.nanmax(np.abs(exact - outs["zero"][sub])) if sol is not None else float("nan")
    print(f"[{name}] {pts.shape[0]} pts, grid {[a.shape for a in arrays32]}, brute-vs-batch {err:.2e}, "
          f"exact-vs-batch {errx:.2e}, "
          f"{time.time() - t0:.1f}s", flush=True)


if __name__ == "__main__":
    names = sys.argv[1:] or sorted(f[: -len(".plan.json")] for f in os.listdir(PLANS) if f.endswith(".plan.json"))
    for i, n in enumerate(names):
        make(n, 2102_08514 + sum(map(ord, n)))
