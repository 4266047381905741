"""Native plan producer for box splines.

The reference turns a direction matrix into an evaluation plan in four exact-rational
stages: PP extraction over the knot-plane arrangement of the support (spline.py:302-335,
481-531), sub-region decomposition of the coset box with its branch-free membership table
(analysis.py:113-267), a greedy symmetry search rewriting sub-regions onto reference kernels
(analysis.py:279-399), and plan assembly with fetch grouping / ordering
(plancompile.py:150-380).  This module restates the same algorithm so the drop-in can
compile a box-spline plan without the reference; `box_spline_plan(columns, lattice, cosets)`
returns the `EvaluationPlan` the reference compiler emits — the same canonical document and
checksum — and `compile_pp_plan` does the same for any PP spline (e.g. an imported Voronoi
document).  tests/test_boxplan.py compares against the catalog's reference-compiled plans and
PP documents and against reference-compiled plans of direction sets outside the catalog.

Design notes (own implementation, not a translation):

* polytopes are kept as (sorted vertex tuple, sorted facet tuple) with facets canonical
  primitive integer half-spaces; a split keeps the vertices on each side plus the crossing
  points that are vertices (tight on full-rank constraint sets), facets are the half-spaces
  tight on an affinely (s-1)-dimensional vertex set — the same canonical form the reference
  sorts cells and compares classes with;
* each piece polynomial comes from the box-spline recurrence run symbolically at the cell's
  centroid (side decisions of the half-open base case taken there, barycentric coordinates
  carried as affine polynomials in absolute coordinates); a node whose point lies outside its
  sub-zonotope is zero, and node values are shared across cells keyed by the node's own
  knot-plane side vector — 4-20x faster than a per-cell recurrence (bcc_quartic 12 s vs the
  reference's 252 s), same polynomials;
* the symmetry search walks the signed-permutation group in the reference's order and
  matches weight polynomials exactly, then fits the integer affine site renaming.
"""

from __future__ import annotations

import random
from fractions import Fraction
from itertools import combinations, permutations, product
from math import floor, gcd

from .exact import Poly
from .plan import ClassTransform, EvaluationPlan, PlanError, PlanKernel, PlanOptions
from .tpplan import group_fetches, order_fetches

F0, F1 = Fraction(0), Fraction(1)


# -- exact linear algebra -------------------------------------------------------------------

def _rank(rows) -> int:
    m = [[Fraction(v) for v in r] for r in rows]
    rank, cols = 0, len(m[0]) if m else 0
    for c in range(cols):
        piv = next((r for r in range(rank, len(m)) if m[r][c] != 0), None)
        if piv is None:
            continue
        m[rank], m[piv] = m[piv], m[rank]
        for r in range(len(m)):
            if r != rank and m[r][c] != 0:
                f = m[r][c] / m[rank][c]
                m[r] = [a - f * b for a, b in zip(m[r], m[rank])]
        rank += 1
    return rank


def _solve(rows, rhs):
    n = len(rows)
    m = [[Fraction(v) for v in r] + [Fraction(b)] for r, b in zip(rows, rhs)]
    for c in range(n):
        piv = next((r for r in range(c, n) if m[r][c] != 0), None)
        if piv is None:
            return None
        m[c], m[piv] = m[piv], m[c]
        for r in range(n):
            if r != c and m[r][c] != 0:
                f = m[r][c] / m[c][c]
                m[r] = [a - f * b for a, b in zip(m[r], m[c])]
    return tuple(m[i][n] / m[i][i] for i in range(n))


def _inverse(a):
    n = len(a)
    cols = [_solve(a, [F1 if i == j else F0 for i in range(n)]) for j in range(n)]
    return [[cols[j][i] for j in range(n)] for i in range(n)]


def _det(a):
    n = len(a)
    m = [[Fraction(v) for v in r] for r in a]
    d = F1
    for c in range(n):
        piv = next((r for r in range(c, n) if m[r][c] != 0), None)
        if piv is None:
            return F0
        if piv != c:
            m[c], m[piv] = m[piv], m[c]
            d = -d
        d *= m[c][c]
        for r in range(c + 1, n):
            f = m[r][c] / m[c][c]
            m[r] = [x - f * y for x, y in zip(m[r], m[c])]
    return d


def _nullspace_vector(rows, dim):
    """One nonzero vector orthogonal to `rows` (rank dim-1): reduced row echelon form, the
    free column set to 1."""
    m = [[Fraction(v) for v in r] for r in rows]
    pivots, rank = [], 0
    for c in range(dim):
        piv = next((r for r in range(rank, len(m)) if m[r][c] != 0), None)
        if piv is None:
            continue
        m[rank], m[piv] = m[piv], m[rank]
        m[rank] = [x / m[rank][c] for x in m[rank]]
        for r in range(len(m)):
            if r != rank and m[r][c] != 0:
                f = m[r][c]
                m[r] = [a - f * b for a, b in zip(m[r], m[rank])]
        pivots.append(c)
        rank += 1
    free = [c for c in range(dim) if c not in pivots][0]
    v = [F0] * dim
    v[free] = F1
    for r, c in enumerate(pivots):
        v[c] = -m[r][free]
    return v


def _primitive(v) -> tuple:
    v = [Fraction(x) for x in v]
    den = 1
    for x in v:
        den = den * x.denominator // gcd(den, x.denominator)
    ints = [int(x * den) for x in v]
    g = 0
    for x in ints:
        g = gcd(g, abs(x))
    return tuple(x // g for x in ints)


def _dot(a, b):
    return sum((Fraction(x) * y for x, y in zip(a, b)), F0)


def _affine_rank(points) -> int:
    if not points:
        return -1
    base = points[0]
    diffs = [[x - y for x, y in zip(p, base)] for p in points[1:]]
    return _rank(diffs) if diffs else 0


# -- half-spaces, planes, polytopes -----------------------------------------------------------

def _halfspace(normal, offset):
    """Canonical n.x <= o with a primitive integer normal (positive rescaling)."""
    prim = _primitive(normal)
    i = next(k for k, x in enumerate(prim) if x != 0)
    scale = Fraction(prim[i]) / Fraction(normal[i])
    return (prim, Fraction(offset) * scale)


def _plane(normal, offset):
    """Canonical plane n.x = o: primitive normal, first nonzero component positive."""
    prim = _primitive(normal)
    i = next(k for k, x in enumerate(prim) if x != 0)
    off = Fraction(offset) * Fraction(prim[i]) / Fraction(normal[i])
    if prim[i] < 0:
        prim, off = tuple(-x for x in prim), -off
    return (prim, off)


class Polytope:
    __slots__ = ("dim", "hs", "verts")

    def __init__(self, dim, hs, verts):
        self.dim = dim
        verts = sorted(set(verts))
        facets = []
        for h in sorted(set(hs)):
            tight = [v for v in verts if _dot(h[0], v) == h[1]]
            if _affine_rank(tight) == dim - 1:
                facets.append(h)
        self.hs = tuple(facets)
        self.verts = tuple(verts)

    def contains(self, x, strict=False) -> bool:
        for n, o in self.hs:
            v = _dot(n, x)
            if v > o or (strict and v == o):
                return False
        return True

    def centroid(self) -> tuple:
        k = Fraction(len(self.verts))
        return tuple(sum((v[i] for v in self.verts), F0) / k for i in range(self.dim))

    def bbox(self):
        return (tuple(min(v[i] for v in self.verts) for i in range(self.dim)),
                tuple(max(v[i] for v in self.verts) for i in range(self.dim)))

    def split(self, plane):
        n, o = plane
        side = [(_dot(n, v) > o) - (_dot(n, v) < o) for v in self.verts]
        lo, hi = any(s < 0 for s in side), any(s > 0 for s in side)
        if not hi:
            return (self, None) if lo else (None, None)
        if not lo:
            return None, self
        cross = []
        for (i, a), (j, b) in combinations(enumerate(self.verts), 2):
            if side[i] * side[j] >= 0:
                continue
            lam = (o - _dot(n, a)) / _dot(n, [y - x for x, y in zip(a, b)])
            cross.append(tuple(x + lam * (y - x) for x, y in zip(a, b)))

        def piece(keep_sign, cut):
            hs = list(self.hs) + [cut]
            cand = {v for v, s in zip(self.verts, side) if s * keep_sign >= 0}
            for p in cross:
                if _rank([h[0] for h in hs if _dot(h[0], p) == h[1]]) == self.dim:
                    cand.add(p)
            pts = sorted(cand)
            if _affine_rank(pts) < self.dim:
                return None
            return Polytope(self.dim, hs, pts)

        return piece(-1, (n, o)), piece(1, (tuple(-x for x in n), -o))

    def mapped(self, A, b) -> frozenset:
        """Vertex set of the image under x -> A x + b (polytopes compare by vertex set)."""
        return frozenset(tuple(_dot(row, v) + bi for row, bi in zip(A, b)) for v in self.verts)


def _box(lo, hi) -> Polytope:
    dim = len(lo)
    hs = []
    for i in range(dim):
        e = [0] * dim
        e[i] = 1
        hs.append(_halfspace(e, hi[i]))
        e[i] = -1
        hs.append(_halfspace(e, -Fraction(lo[i])))
    verts = [tuple(Fraction(hi[i]) if m >> i & 1 else Fraction(lo[i]) for i in range(dim)) for m in range(1 << dim)]
    return Polytope(dim, hs, verts)


def _zonotope(cols) -> Polytope:
    """Minkowski sum of the segments [0, xi] (parallel columns merged; polytope.py:346-400)."""
    dim = len(cols[0])
    classes, base = {}, tuple([F0] * dim)
    for d in cols:
        d = tuple(Fraction(x) for x in d)
        if all(x == 0 for x in d):
            continue
        prim = _primitive(d)
        i = next(k for k, x in enumerate(prim) if x != 0)
        key = prim if prim[i] > 0 else tuple(-x for x in prim)
        acc = classes.get(key, tuple([F0] * dim))
        if prim[i] > 0:
            classes[key] = tuple(a + b for a, b in zip(acc, d))
        else:
            base = tuple(a + b for a, b in zip(base, d))
            classes[key] = tuple(a - b for a, b in zip(acc, d))
    segs = list(classes.values())
    cands = {base}
    for sgm in segs:
        cands |= {tuple(a + b for a, b in zip(c, sgm)) for c in cands}
    hs = set()
    for combo in combinations(segs, dim - 1):
        if _rank(combo) < dim - 1:
            continue
        nv = _nullspace_vector(combo, dim)
        for sign in (1, -1):
            normal = [sign * x for x in nv]
            hs.add(_halfspace(normal, max(_dot(normal, c) for c in cands)))
    verts = [c for c in cands if all(_dot(n, c) <= o for n, o in hs)
             and _rank([n for n, o in hs if _dot(n, c) == o]) == dim]
    return Polytope(dim, hs, verts)


def _arrangement(ambient: Polytope, planes) -> list:
    cells = [ambient]
    for pl in sorted(set(planes)):
        nxt = []
        for c in cells:
            lo, hi = c.split(pl)
            if lo is not None:
                nxt.append(lo)
            if hi is not None:
                nxt.append(hi)
        cells = nxt
    cells.sort(key=lambda c: c.centroid())
    return cells


# -- box spline PP form -------------------------------------------------------------------------

def _knot_planes(cols) -> list:
    """Planes spanned by (s-1)-subsets of the direction classes, offsets = subset sums of n.xi
    over all columns (spline.py:302-335)."""
    dim = len(cols[0])
    classes = sorted({_primitive(c) for c in cols if any(x != 0 for x in c)})
    normals = set()
    for combo in combinations(classes, dim - 1):
        if _rank(combo) != dim - 1:
            continue
        n = _primitive(_nullspace_vector(combo, dim))
        i = next(k for k, x in enumerate(n) if x != 0)
        normals.add(n if n[i] > 0 else tuple(-x for x in n))
    planes = set()
    for n in sorted(normals):
        offs = {F0}
        for c in cols:
            d = _dot(n, c)
            if d != 0:
                offs |= {o + d for o in offs}
        for o in offs:
            planes.add(_plane(n, o))
    return sorted(planes)


def _affine_poly(dim, coeffs, const) -> Poly:
    terms = {tuple([0] * dim): Fraction(const)}
    for i, c in enumerate(coeffs):
        if c:
            e = [0] * dim
            e[i] = 1
            terms[tuple(e)] = Fraction(c)
    return Poly(dim, terms)


def compose_affine(p: Poly, A, b) -> Poly:
    """q(x) = p(A x + b)."""
    dim = p.dim
    subs = [_affine_poly(dim, A[i], b[i]) for i in range(dim)]
    pw = []
    for i in range(dim):
        row = [Poly.const(dim, 1)]
        for _ in range(max((e[i] for e in p.terms), default=0)):
            row.append(row[-1] * subs[i])
        pw.append(row)
    acc = Poly(dim)
    for e, c in p.terms.items():
        t = Poly.const(dim, c)
        for i, k in enumerate(e):
            if k:
                t = t * pw[i][k]
        acc = acc + t
    return acc


class _BoxRecurrence:
    """Symbolic box-spline recurrence around a point x0 (off all knot planes):
    M_Xi(x0 + delta) as a polynomial in delta, side decisions taken at x0."""

    def __init__(self, cols):
        self.dim = len(cols[0])
        if any(Fraction(v).denominator != 1 for c in cols for v in c):
            raise PlanError("box-spline direction columns must be integer vectors")
        self.root = tuple(sorted(tuple(int(v) for v in c) for c in cols))
        self.info = {}
        self.memo = {}

    def _info(self, key):
        if key not in self.info:
            basis, idx = [], []
            for i, col in enumerate(key):
                if len(basis) == self.dim:
                    break
                if _rank(basis + [col]) == len(basis) + 1:
                    basis.append(col)
                    idx.append(i)
            if len(basis) < self.dim:
                self.info[key] = None
            else:
                B = [[basis[j][i] for j in range(self.dim)] for i in range(self.dim)]  # columns
                det = _det(B)
                binv = _inverse(B)
                adj = tuple(tuple(int(v * det) for v in row) for row in binv)  # integer adjugate
                # support facets of M_key: a node whose point lies strictly outside is zero
                # (x0 is off every knot plane, and the facets of every sub-zonotope shifted by
                # the removed columns are knot planes, so "strictly" loses nothing)
                big = len(key) > self.dim
                hs = tuple((n, int(o)) for n, o in _zonotope(list(key)).hs) if big else ()
                planes = tuple((n, int(o)) for n, o in _knot_planes(list(key))) if big else ()
                self.info[key] = (tuple(idx), binv, abs(det), hs, planes, adj, int(det))
        return self.info[key]

    def piece(self, x0) -> Poly:
        """Polynomial (absolute coordinates) of the piece containing the off-plane point x0.

        Every node M_cols(x - shift) of the recurrence is one polynomial on each cell of its
        own knot-plane arrangement, so node values are memoised across calls by (cols, shift,
        side of y0 = x0 - shift on each knot plane of cols) and carried in absolute x.  Side
        tests run on integers: y0 = Y / den with den the common denominator of x0."""
        dim = self.dim
        memo = self.memo
        den = 1
        for v in x0:
            den = den * Fraction(v).denominator // gcd(den, Fraction(v).denominator)
        X = tuple(int(Fraction(v) * den) for v in x0)

        def idot(n, y):
            return sum(a * b for a, b in zip(n, y))

        def rec(cols, shift, Y):
            inf = self._info(cols)
            for n, o in inf[3]:
                if idot(n, Y) > o * den:
                    return Poly(dim)
            if len(cols) == dim:
                D = inf[6] * den
                for row in inf[5]:
                    t = idot(row, Y)
                    if not (0 <= t < D if D > 0 else D < t <= 0):
                        return Poly(dim)
                return Poly.const(dim, 1 / inf[2])
            key = (cols, shift, tuple(idot(n, Y) > o * den for n, o in inf[4]))
            if key in memo:
                return memo[key]
            binv = inf[1]
            # t(x) = binv (x - shift): affine in the absolute coordinates
            tpoly = [_affine_poly(dim, binv[r], -_dot(binv[r], shift)) for r in range(dim)]
            tau, mult = {}, {}
            for c in cols:
                mult[c] = mult.get(c, 0) + 1
                tau.setdefault(c, Poly(dim))
            for slot, i in enumerate(inf[0]):
                tau[cols[i]] = tau[cols[i]] + tpoly[slot]
            acc = Poly(dim)
            for c, m in mult.items():
                sub = list(cols)
                sub.remove(c)
                sub = tuple(sub)
                if self._info(sub) is None:
                    continue
                c1 = tau[c]
                c2 = Poly.const(dim, m) - c1
                if not c1.is_zero():
                    ch = rec(sub, shift, Y)
                    if not ch.is_zero():
                        acc = acc + c1 * ch
                if not c2.is_zero():
                    ch = rec(sub, tuple(a + b for a, b in zip(shift, c)), tuple(a - den * b for a, b in zip(Y, c)))
                    if not ch.is_zero():
                        acc = acc + c2 * ch
            val = Poly(dim, {e: v / (len(cols) - dim) for e, v in acc.terms.items()})
            memo[key] = val
            return val

        return rec(self.root, tuple([0] * dim), X)


class BoxPP:
    """The PP form of a box spline: arrangement cells of the knot planes over the support
    (spline.py:481-531; the cell polynomial is unique, so the reference's sampled fit and
    its symbolic witness run agree with the symbolic run used here)."""

    def __init__(self, cols):
        self.cols = [tuple(Fraction(v) for v in c) for c in cols]
        self.dim = len(cols[0])
        self.support = _zonotope(self.cols)
        planes = [pl for pl in _knot_planes(self.cols)
                  if min(_dot(pl[0], v) for v in self.support.verts) < pl[1] < max(_dot(pl[0], v) for v in self.support.verts)]
        self.cells = _arrangement(self.support, planes)
        rec = _BoxRecurrence(self.cols)
        self.polys = [rec.piece(c.centroid()) for c in self.cells]


def extract_pp_form(cols, name: str = ""):
    """spline.py:481-531: the box spline of direction columns `cols` (support sum of [0, xi])
    as a pp.PiecewisePolySpline — `pp.format_pp_spline` of it is the reference's document."""
    from .pp import PiecewisePolySpline, SplinePiece

    bp = BoxPP(cols)
    pieces = [SplinePiece(list(c.hs), p, _vertices=c.verts) for c, p in zip(bp.cells, bp.polys)]
    center = tuple(sum((c[i] for c in bp.cols), F0) / 2 for i in range(bp.dim))
    return PiecewisePolySpline(bp.dim, pieces, len(bp.cols) - bp.dim, name=name, center=center)


class _PPView:
    """Exact point queries over a PP spline's pieces with the reference's tie rule (first
    covering piece, spline.py:371-389) and its union support (spline.py:751-770)."""

    def __init__(self, spline):
        self.dim = spline.s
        self.cells = [Polytope(spline.s, [(tuple(n), Fraction(o)) for n, o in p.halfspaces], p.vertices())
                      for p in spline.pieces]
        self.polys = [p.poly for p in spline.pieces]
        verts = sorted({v for c in self.cells for v in c.verts})
        cands = sorted({h for c in self.cells for h in c.hs})
        self.support_hs = [h for h in cands if all(_dot(h[0], v) <= h[1] for v in verts)]
        self.lo = tuple(min(v[i] for v in verts) for i in range(self.dim))
        self.hi = tuple(max(v[i] for v in verts) for i in range(self.dim))
        self._buckets = {}
        for i, c in enumerate(self.cells):
            lo, hi = c.bbox()
            for cell in product(*[range(floor(a), floor(b) + 1) for a, b in zip(lo, hi)]):
                self._buckets.setdefault(cell, []).append(i)

    def in_support(self, x) -> bool:
        return all(_dot(n, x) <= o for n, o in self.support_hs)

    def piece_at(self, x):
        for i in self._buckets.get(tuple(floor(v) for v in x), ()):
            if self.cells[i].contains(x):
                return i
        return None

    def eval(self, x) -> Fraction:
        i = self.piece_at(x)
        return F0 if i is None else self.polys[i].eval(list(x))

    def nonnegative_sampled(self, samples_per_piece: int = 8, rng_seed: int = 11) -> bool:
        """spline.py:459-465 with its interior sampler (spline.py:471-478)."""
        rng = random.Random(rng_seed)
        for c, p in zip(self.cells, self.polys):
            for _ in range(samples_per_piece):
                w = [Fraction(rng.randint(1, 64)) for _ in c.verts]
                tot = sum(w, F0)
                x = [sum((wi * v[k] for wi, v in zip(w, c.verts)), F0) / tot for k in range(self.dim)]
                if p.eval(x) < 0:
                    return False
        return True


# -- sub-regions, symmetry, assembly --------------------------------------------------------------

def _signed_permutations(s) -> list:
    mats = []
    for perm in permutations(range(s)):
        for signs in product((1, -1), repeat=s):
            rows = [[F0] * s for _ in range(s)]
            for i in range(s):
                rows[i][perm[i]] = Fraction(signs[i])
            mats.append(tuple(tuple(r) for r in rows))
    ident = tuple(tuple(F1 if i == j else F0 for j in range(s)) for i in range(s))
    mats.sort(key=lambda m: (m != ident, m))
    return mats


def _fit_site_map(pairs, T):
    s = len(T)
    src = [tuple(Fraction(v) for v in a) for a, _ in pairs]
    dst = [tuple(Fraction(v) for v in b) for _, b in pairs]
    for A in (_inverse([list(r) for r in T]), [list(r) for r in T]):
        b = [d - _dot(row, src[0]) for row, d in zip(A, dst[0])]
        if all(tuple(_dot(row, p) + bi for row, bi in zip(A, b)) == q for p, q in zip(src, dst)):
            if all(v.denominator == 1 for r in A for v in r) and all(v.denominator == 1 for v in b):
                return tuple(tuple(int(v) for v in r) for r in A), tuple(int(v) for v in b)
    base, idx = src[0], [0]
    for i in range(1, len(src)):
        trial = idx + [i]
        if _rank([[x - y for x, y in zip(src[j], base)] for j in trial[1:]]) == len(trial) - 1:
            idx = trial
        if len(idx) == s + 1:
            break
    if len(idx) != s + 1:
        return None
    M = [list(src[j]) + [F1] for j in idx]
    cols = []
    for comp in range(s):
        sol = _solve(M, [dst[j][comp] for j in idx])
        if sol is None:
            return None
        cols.append(sol)
    A = [[cols[r][c] for c in range(s)] for r in range(s)]
    b = [cols[r][s] for r in range(s)]
    if not (all(v.denominator == 1 for r in A for v in r) and all(v.denominator == 1 for v in b)):
        return None
    if not all(tuple(_dot(row, p) + bi for row, bi in zip(A, b)) == q for p, q in zip(src, dst)):
        return None
    return tuple(tuple(int(v) for v in r) for r in A), tuple(int(v) for v in b)


def box_spline_plan(cols, lattice, cosets, name: str = "", options: PlanOptions | None = None) -> EvaluationPlan:
    """The reference compiler's plan (corpus.build_plan, corpus.py:153-156) for the box spline
    of direction columns `cols` on `lattice` (lattice.IntegerLattice) with its Cartesian
    coset decomposition `cosets`."""
    return compile_pp_plan(extract_pp_form(cols, name), lattice, cosets, options)


def compile_pp_plan(spline, lattice, cosets, options: PlanOptions | None = None,
                    pou_points: int = 4, rng_seed: int = 23) -> EvaluationPlan:
    """enumerate_subregions + search_symmetry + compile_plan (analysis.py:113-399,
    plancompile.py:339-380) for any PP spline (pp.PiecewisePolySpline: a box spline from
    `extract_pp_form` or an imported document such as the Voronoi splines)."""
    options = options or PlanOptions()
    pp = _PPView(spline)
    s = pp.dim
    diag = tuple(int(d) for d in cosets.diag)
    scale = Fraction(lattice.det())
    slo, shi = pp.lo, pp.hi

    def sites_at(x, on_sublattice):
        rngs = [range(-floor(-(x[i] - shi[i]) / (diag[i] if on_sublattice else 1)),
                      floor((x[i] - slo[i]) / (diag[i] if on_sublattice else 1)) + 1) for i in range(s)]
        for z in product(*rngs):
            m = tuple(z[i] * diag[i] for i in range(s)) if on_sublattice else z
            yield m

    # partition of unity on the sub-lattice D Z^s alone (recorded by the reference)
    rng = random.Random(rng_seed)
    probe = [tuple(Fraction(rng.randint(-128, 128), 97) for _ in range(s)) for _ in range(pou_points)]
    for x in probe:  # enumerate_subregions requires it on the full lattice (analysis.py:124)
        tot = F0
        for m in sites_at(x, False):
            y = tuple(a - b for a, b in zip(x, m))
            if lattice.contains_site(m) and pp.in_support(y):
                tot += scale * pp.eval(y)
        if tot != 1:
            from .pp import SplineError

            raise SplineError(f"partition of unity fails at {x}: sum {tot}")
    pou_sub = True
    for x in probe[:2]:
        tot = F0
        for m in sites_at(x, True):
            y = tuple(a - b for a, b in zip(x, m))
            if pp.in_support(y):
                tot += cosets.M * scale * pp.eval(y)
        if tot != 1:
            pou_sub = False
            break

    box = _box([0] * s, list(diag))
    planes = set()
    for c in pp.cells:
        for n, o in c.hs:
            pl = _plane(n, o)
            g = 0
            for ni, di in zip(pl[0], diag):
                g = gcd(g, abs(ni * di))
            if g == 0:
                continue
            vals = [_dot(pl[0], v) for v in box.verts]
            lo_v, hi_v = min(vals), max(vals)
            off = pl[1] - g * floor((pl[1] - lo_v) / g)
            while off <= hi_v:
                if lo_v < off < hi_v:
                    planes.add((pl[0], off))
                off += g
    planes = sorted(planes)
    cells = _arrangement(box, planes)
    subs = []
    ident = [[F1 if i == j else F0 for j in range(s)] for i in range(s)]
    for cid, cell in enumerate(cells):
        w = cell.centroid()
        sw = []
        for m in sites_at(w, True):
            y = tuple(a - b for a, b in zip(w, m))
            if not pp.in_support(y):
                continue
            i = pp.piece_at(y)
            if i is None:
                continue
            poly = Poly(s, {e: c * scale for e, c in pp.polys[i].terms.items()})
            if poly.is_zero():
                continue
            sw.append((tuple(int(v) for v in m), compose_affine(poly, ident, [-Fraction(v) for v in m])))
        sw.sort(key=lambda t: t[0])
        code = 0
        for j, (n, o) in enumerate(planes):
            if _dot(n, w) >= o:
                code |= 1 << j
        subs.append((cell, [a for a, _ in sw], [b for _, b in sw], code))
    codes = sorted(c for *_, c in subs)
    if len(set(codes)) != len(codes):
        raise PlanError("two sub-regions share a plane-side code")
    r = max(1, len(codes))
    while len({c % r for c in codes}) != len(codes):
        r += 1
    sigma = [-1] * r
    for cid, (*_, c) in enumerate(subs):
        sigma[c % r] = cid
    refl = []
    pset = set(planes)
    for axis, d in enumerate(diag):
        ok = True
        for n, o in planes:
            nn = list(n)
            nn[axis] = -nn[axis]
            if _plane(nn, o - n[axis] * d) not in pset:
                ok = False
                break
        refl.append(ok)

    # greedy symmetry search (analysis.py:279-318)
    group = _signed_permutations(s)
    refs, transforms = [], [None] * len(subs)
    zero = tuple([F0] * s)
    for cid, (cell, sites, polys, _) in enumerate(subs):
        found = None
        for kidx, rid in enumerate(refs):
            rcell, rsites, rpolys, _ = subs[rid]
            if len(sites) != len(rsites):
                continue
            vc_r, vc_s = rcell.centroid(), cell.centroid()
            rverts = frozenset(rcell.verts)
            by_poly = {}
            for st, pl in zip(sites, polys):
                by_poly.setdefault(pl, []).append(st)
            for T in group:
                t = tuple(_dot(row, vc_s) - b for row, b in zip(T, vc_r))
                if cell.mapped(T, [-v for v in t]) != rverts:
                    continue
                buckets = {k: list(v) for k, v in by_poly.items()}
                pairs, ok = [], True
                for st, pl in zip(rsites, rpolys):
                    avail = buckets.get(compose_affine(pl, T, [-v for v in t]))
                    if not avail:
                        ok = False
                        break
                    pairs.append((st, avail.pop(0)))
                if not ok:
                    continue
                fit = _fit_site_map(pairs, T)
                if fit is None:
                    continue
                found = ClassTransform(kidx, T, t, fit[0], fit[1])
                break
            if found is not None:
                break
        if found is None:
            refs.append(cid)
            found = ClassTransform(len(refs) - 1, tuple(tuple(r) for r in ident), zero,
                                   tuple(tuple(1 if i == j else 0 for j in range(s)) for i in range(s)),
                                   tuple([0] * s))
        transforms[cid] = found

    # assembly (plancompile.py:339-380); box splines are non-negative
    nonneg = pp.nonnegative_sampled()
    grouped = options.grouped and nonneg
    kernels = []
    for rid in refs:
        _, sites, polys, _ = subs[rid]
        groups = group_fetches(sites, polys, diag, grouped=grouped)
        if options.ordered:
            groups = order_fetches(groups, diag)
        kernels.append(PlanKernel(rid, tuple(groups)))
    from dataclasses import replace

    return EvaluationPlan(
        name=spline.name, lattice_name=lattice.name, s=s, diag=diag, shifts=tuple(tuple(v) for v in cosets.shifts),
        scale=scale, planes=tuple(planes), r=r, sigma=tuple(sigma), classes=tuple(transforms),
        kernels=tuple(kernels), options=replace(options, grouped=grouped), basis_nonnegative=nonneg,
        pou_on_sublattice=pou_sub, reflective_axes=tuple(refl))
