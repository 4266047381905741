"""Piecewise-polynomial (PP) descriptions of the Voronoi splines V1 on FCC and BCC.

Build-container tool (needs /root/reference).  The reference declares Voronoi-spline
construction out of scope and only IMPORTS externally supplied PP data
(`SPEC.md:8`, `spline.py:667-713`).  This script supplies that data,
built only from the reference's own exact tools, following the paper's construction
(`PAPER.md:154-159`):

  * V0 = chi_L / |det L| on the Voronoi cell.  The Voronoi cell of FCC (rhombic
    dodecahedron) and of BCC (truncated octahedron) is a centred zonotope
    Z(g_1..g_n); a fine zonotopal tiling (lower faces of a generic lift) writes
    chi_Z = sum_B |det B| * M_B(x - s_B) over the bases B of the generators, so V0
    is a sum of 4 (FCC) or 16 (BCC) constant box splines.
  * V1 = V0 * V0 = sum_{B,C} |det B||det C| / vol^2 * M_{B u C}(x - s_B - s_C):
    16 (FCC) / 256 (BCC) shifted 6-direction box splines (M_A * M_B = M_{A u B}).
  * Each distinct 6-direction box spline is extracted with the reference's
    `extract_pp_form` (`spline.py:481-531`, holdout-verified against the exact
    recurrence `boxspline_eval_exact`, `spline.py:144-207`).
  * The union of the terms' shifted knot planes (`harvest_knot_planes`,
    `spline.py:302-335`) cuts the support (2x the Voronoi cell) into an arrangement
    (`build_arrangement`, `polytope.py:421-442`); per cell, the polynomial is the sum of
    the terms' pieces, composed with their shifts.  Planes across which no cell pair
    changes polynomial are dropped and the arrangement rebuilt.
  * Checks: V0's tiling volume equals the cell volume and V0 equals the indicator at
    random points; V1 per cell equals sum of `boxspline_eval_exact` at random interior
    points AND the geometric definition vol(Z n (x - Z)) / vol(Z)^2 (an independent
    exact evaluator); then `import_pp_spline(format_pp_spline(sp), validate=True)`
    (tiling, unit integral, facet continuity, non-negativity; `spline.py:412-457`).

Output: tests/golden/voronoi/<name>.spp (the reference's import format).

usage: python tools/voronoi_pp.py fcc_voronoi1|bcc_voronoi1 [--jobs J]
"""
from __future__ import annotations

import os
import random
import sys
import time
from itertools import combinations

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from refshim import import_reference  # noqa: E402

import_reference()
from splineplan.exactmath import R0, RationalMatrix, poly_compose_affine, rat, vadd, vdot, vec, vsub  # noqa: E402
from splineplan.polytope import ConvexPolytope, HalfSpace, Plane, build_arrangement, minkowski_sum_segments  # noqa: E402
from splineplan.spline import (  # noqa: E402
    DirectionMatrix,
    PiecewisePolySpline,
    SplinePiece,
    boxspline_eval_exact,
    extract_pp_form,
    format_pp_spline,
    harvest_knot_planes,
    import_pp_spline,
)

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT_DIR = os.path.join(REPO, "tests", "golden", "voronoi")

H = rat(1, 2)
# Voronoi cells as centred zonotopes sum_i [-g_i/2, g_i/2].
GENERATORS = {
    # FCC (even coordinate sum; lattice.py:_NAMED["FCC"]): rhombic dodecahedron,
    # vertices (+-1,0,0)-type and (+-1/2,+-1/2,+-1/2): the 4 body diagonals / 2.
    "fcc": [(1, 1, 1), (-1, 1, 1), (1, -1, 1), (1, 1, -1)],
    # BCC (all-even or all-odd): truncated octahedron, vertices perms of (+-1,+-1/2,0):
    # the 6 face diagonals / 2.
    "bcc": [(1, 1, 0), (1, -1, 0), (1, 0, 1), (1, 0, -1), (0, 1, 1), (0, 1, -1)],
}
LATTICE = {"fcc": "FCC", "bcc": "BCC"}


def gens_of(kind):
    return [tuple(H * c for c in g) for g in GENERATORS[kind]]


def centred_zonotope(gens):
    z = minkowski_sum_segments(gens)
    half = tuple(-sum((g[i] for g in gens), R0) / 2 for i in range(3))
    return z.translated(half)


def voronoi_cell(kind):
    """Voronoi region of the origin from the lattice's short vectors (independent of
    the zonotope description)."""
    from splineplan.lattice import named_lattice

    lat = named_lattice(LATTICE[kind])
    hs = []
    rng = range(-2, 3)
    for p in ((a, b, c) for a in rng for b in rng for c in rng):
        if p == (0, 0, 0) or not lat.contains_site(p):
            continue
        hs.append(HalfSpace.make(p, rat(vdot(p, p), 2)))
    return ConvexPolytope.from_halfspaces(hs, 3)


def zonotope_tiling(gens, seed=5):
    """Fine tiling of Z(gens) (non-centred sum [0, g]) into parallelepipeds: the
    lower facets of the lift g -> (g, h_g) with generic heights.  Returns
    [(basis columns, shift)]."""
    rnd = random.Random(seed)
    heights = [rat(rnd.randint(1, 10**6), 997) for _ in gens]
    tiles = []
    for B in combinations(range(len(gens)), 3):
        M = RationalMatrix([gens[i] for i in B])      # rows = generators
        if M.rank() < 3:
            continue
        w = M.solve([-heights[i] for i in B])          # <w, g_i> = -h_i on B
        shift = (R0, R0, R0)
        for j in range(len(gens)):
            if j in B:
                continue
            v = vdot(w, gens[j]) + heights[j]
            if v == 0:
                raise RuntimeError("non-generic heights")
            if v < 0:
                shift = vadd(shift, gens[j])
        tiles.append(([gens[i] for i in B], shift))
    return tiles


def basis_det(cols):
    return abs(RationalMatrix.from_columns(cols).det())


def v0_terms(kind):
    gens = gens_of(kind)
    Z = centred_zonotope(gens)
    vol = Z.volume()
    centre = tuple(-sum((g[i] for g in gens), R0) / 2 for i in range(3))
    terms = []
    for cols, shift in zonotope_tiling(gens):
        # 1_P(x) = |det B| * M_B(x - shift_P);  V0 = 1_Z / vol
        terms.append((tuple(sorted(cols)), vadd(shift, centre), basis_det(cols) / vol))
    return Z, vol, terms


def v1_terms(kind):
    Z, vol, t0 = v0_terms(kind)
    acc = {}
    for (ca, sa, wa) in t0:
        for (cb, sb, wb) in t0:
            key = (tuple(sorted(ca + cb)), vadd(sa, sb))
            acc[key] = acc.get(key, R0) + wa * wb
    return Z, vol, t0, [(cols, shift, w) for (cols, shift), w in sorted(acc.items())]


def check_v0(kind, Z, vol, t0, samples=300):
    vor = voronoi_cell(kind)
    assert sorted(vor.halfspaces) == sorted(Z.halfspaces), "zonotope != Voronoi cell"
    assert sum(basis_det(c) for c, _, _ in t0) == vol, "tiling volume"
    from splineplan.lattice import named_lattice

    assert vol == named_lattice(LATTICE[kind]).det()
    rnd = random.Random(1)
    for _ in range(samples):
        x = tuple(rat(rnd.randint(-1500, 1500), 1009) for _ in range(3))
        v = sum((w * boxspline_eval_exact(DirectionMatrix(c), vsub(x, s)) for c, s, w in t0), R0)
        expect = 1 / vol if Z.contains(x, strict=True) else R0
        if not Z.contains(x) or Z.contains(x, strict=True):
            assert v == expect, (x, v, expect)


def _extract(cols):
    t = time.time()
    sp = extract_pp_form(DirectionMatrix(list(cols)))
    return cols, sp, time.time() - t


def support_of(Z):
    verts = [tuple(2 * v for v in p) for p in Z.vertices]
    hs = [HalfSpace(h.normal, 2 * h.offset) for h in Z.halfspaces]
    return ConvexPolytope(3, tuple(sorted(hs)), tuple(sorted(verts)))


def geometric_v1(Z, vol, x):
    """vol(Z n (x - Z)) / vol^2 = (chi_Z * chi_Z)(x) / vol^2 (Z is centrally symmetric)."""
    hs = list(Z.halfspaces) + [HalfSpace(h.normal, h.offset + vdot(h.normal, x)) for h in Z.halfspaces]
    try:
        P = ConvexPolytope.from_halfspaces(hs, 3)
    except Exception:
        return R0
    return P.volume() / (vol * vol)


def build(kind, jobs=8, log=print):
    t_start = time.time()
    Z, vol, t0, t1 = v1_terms(kind)
    log(f"[{kind}] V0: {len(t0)} box splines, V1: {len(t1)} shifted terms, "
        f"{len({c for c, _, _ in t1})} distinct direction sets")
    check_v0(kind, Z, vol, t0)
    log(f"[{kind}] V0 tiling checked ({time.time()-t_start:.1f}s)")

    distinct = sorted({c for c, _, _ in t1})
    pps = {}
    if jobs > 1:
        from multiprocessing import Pool

        with Pool(jobs) as pool:
            for cols, sp, dt in pool.imap_unordered(_extract, distinct):
                pps[cols] = sp
                log(f"[{kind}]   extracted {len(sp.pieces)} pieces in {dt:.1f}s ({len(pps)}/{len(distinct)})")
    else:
        for cols in distinct:
            cols, sp, dt = _extract(cols)
            pps[cols] = sp
    log(f"[{kind}] extraction done ({time.time()-t_start:.1f}s)")

    support = support_of(Z)
    planes = set()
    for cols, shift, _ in t1:
        for p in pps[cols].pieces:
            for h in p.region.halfspaces:
                planes.add(Plane.make(h.normal, h.offset + vdot(h.normal, shift)))
    planes = sorted(p for p in planes if _meets_interior(p, support))
    log(f"[{kind}] {len(planes)} candidate knot planes")

    def cell_poly(w):
        acc = None
        for cols, shift, wt in t1:
            sp = pps[cols]
            i = sp.piece_at(vsub(w, shift))
            if i is None:
                continue
            p = poly_compose_affine(sp.pieces[i].poly, RationalMatrix.identity(3), tuple(-v for v in shift)).scaled(wt)
            acc = p if acc is None else acc + p
        return acc

    arr = build_arrangement(support, planes)
    polys = [cell_poly(w) for w in arr.witnesses]
    log(f"[{kind}] full arrangement: {len(arr.cells)} cells ({time.time()-t_start:.1f}s)")

    needed = set()
    for ci, cell in enumerate(arr.cells):
        for h in cell.halfspaces:
            pl = Plane.make(h.normal, h.offset)
            if pl not in planes or pl in needed:
                continue
            tight = [v for v in cell.vertices if h.slack(v) == 0]
            fc = tuple(sum(col, R0) / len(tight) for col in zip(*tight))
            eps = rat(1, 1 << 20)
            q = vadd(fc, tuple(eps * n for n in h.normal))      # just outside this cell
            if not support.contains(q, strict=True):
                continue
            j = arr.locate(q)
            if j is not None and j != ci and polys[j] != polys[ci]:
                needed.add(pl)
    planes2 = sorted(needed)
    arr2 = build_arrangement(support, planes2)
    pieces = []
    for cell, w in zip(arr2.cells, arr2.witnesses):
        p = cell_poly(w)
        pieces.append(SplinePiece(cell, p))
    log(f"[{kind}] {len(planes2)} knot planes kept -> {len(pieces)} pieces ({time.time()-t_start:.1f}s)")

    # independent checks at random interior points of every piece
    rnd = random.Random(3)
    for k, pc in enumerate(pieces):
        for _ in range(2):
            wts = [rat(rnd.randint(1, 64)) for _ in pc.region.vertices]
            tot = sum(wts, R0)
            x = tuple(sum((wv * v[i] for wv, v in zip(wts, pc.region.vertices)), R0) / tot for i in range(3))
            val = pc.poly.eval(x)
            bs = sum((wt * boxspline_eval_exact(DirectionMatrix(list(c)), vsub(x, s)) for c, s, wt in t1), R0)
            assert val == bs, ("box-spline sum mismatch", k, x)
            if k % 4 == 0:
                assert val == geometric_v1(Z, vol, x), ("geometric mismatch", k, x)
    log(f"[{kind}] pieces agree with the box-spline sum and the geometric definition ({time.time()-t_start:.1f}s)")

    deg = max(p.poly.degree() for p in pieces)
    name = f"{kind}_voronoi1"
    sp = PiecewisePolySpline(3, pieces, support, deg, name=name, center=(R0, R0, R0))
    text = format_pp_spline(sp)
    sp2 = import_pp_spline(text, validate=True)
    assert len(sp2.pieces) == len(pieces)
    log(f"[{kind}] import_pp_spline(validate=True) passed ({time.time()-t_start:.1f}s)")
    os.makedirs(OUT_DIR, exist_ok=True)
    with open(os.path.join(OUT_DIR, f"{name}.spp"), "w") as fh:
        fh.write(text)
    return sp2


def _meets_interior(plane, poly):
    vals = [vdot(plane.normal, v) for v in poly.vertices]
    return min(vals) < plane.offset < max(vals)


if __name__ == "__main__":
    jobs = 8
    if "--jobs" in sys.argv:
        jobs = int(sys.argv[sys.argv.index("--jobs") + 1])
    for a in sys.argv[1:]:
        if a.endswith("_voronoi1"):
            build(a.split("_")[0], jobs=jobs, log=lambda m: print(m, flush=True))
