"""Piecewise-polynomial spline descriptions: the spline-selection side of the drop-in.

The reference's `corpus.build_spline` / `build_pair` (corpus.py:124-144) return the PP form
of a named spline (`PiecewisePolySpline`, spline.py:344-469) and its pairing with a lattice
(`SplineOnLattice`, spline.py:576-637); PP forms travel as `.spp` text documents
(`format_pp_spline` / `import_pp_spline`, spline.py:645-713), which is also the reference's
cache format.  The drop-in ships the documents of its catalog splines
(`paper_2102_08514_b200/pp/*.spp`, made by the reference's own `extract_pp_form`,
tools/gen_pp.py; the Voronoi ones by tools/voronoi_pp.py) and restates the parts a caller
uses on the host: parsing / formatting (same document text), exact point queries
(`piece_at`, `eval_exact`, `eval_float`), the lattice pairing with its |det L| scale,
contributing sites and partition of unity.  `validate()` runs the structural checks that
need no polytope volumes (declared degree bound, bounded pieces, exact partition of unity on
the lattice and non-negativity at sampled points); the full tiling / unit-integral /
facet-continuity validation stays the reference's (spline.py:412-457), which produced and
validated every shipped document.  Evaluation at scale is the GPU's (`PlanInterpreter`).
"""

from __future__ import annotations

import random
from dataclasses import dataclass, field
from fractions import Fraction
from itertools import combinations, product
from math import floor
from typing import Sequence

from .exact import Poly, frac, frac_str

MAGIC = "splinepp"
VERSION = "1"


class SplineError(ValueError):
    pass


def _solve(rows, rhs):
    """Exact solution of a square system (Gauss-Jordan on Fractions), or None if singular."""
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


@dataclass
class SplinePiece:
    """Region {x : n.x <= o for every half-space (n, o)} and its polynomial."""

    halfspaces: list
    poly: Poly
    _vertices: tuple | None = field(default=None, repr=False)

    def contains(self, x: Sequence, strict: bool = False) -> bool:
        for n, o in self.halfspaces:
            v = sum(Fraction(ni) * xi for ni, xi in zip(n, x))
            if v > o or (strict and v == o):
                return False
        return True

    def vertices(self) -> tuple:
        """Vertex enumeration: feasible intersections of `dim` half-space boundaries."""
        if self._vertices is None:
            dim = len(self.halfspaces[0][0])
            vs = set()
            for h in combinations(self.halfspaces, dim):
                p = _solve([n for n, _ in h], [o for _, o in h])
                if p is not None and self.contains(p):
                    vs.add(p)
            if not vs:
                raise SplineError("empty or unbounded piece")
            self._vertices = tuple(sorted(vs))
        return self._vertices

    def bbox(self) -> tuple:
        vs = self.vertices()
        return (tuple(min(v[i] for v in vs) for i in range(len(vs[0]))),
                tuple(max(v[i] for v in vs) for i in range(len(vs[0]))))


class PiecewisePolySpline:
    """spline.py:344-469: pieces tiling a convex support; a point query resolves boundary
    ties to the first covering piece (adjacent pieces agree there)."""

    def __init__(self, s: int, pieces: Sequence[SplinePiece], degree_bound: int, name: str = "", center=None):
        self.s = s
        self.pieces = tuple(pieces)
        self.degree_bound = int(degree_bound)
        self.name = name
        self.center = tuple(Fraction(c) for c in center) if center is not None else None

    def piece_at(self, x: Sequence):
        x = [Fraction(v) for v in x]
        for i, p in enumerate(self.pieces):
            if p.contains(x):
                return i
        return None

    def eval_exact(self, x: Sequence) -> Fraction:
        i = self.piece_at(x)
        return Fraction(0) if i is None else self.pieces[i].poly.eval([Fraction(v) for v in x])

    def eval_float(self, x: Sequence[float]) -> float:
        i = self.piece_at([Fraction(v) for v in x])
        return 0.0 if i is None else self.pieces[i].poly.eval_float([float(v) for v in x])

    def support_bbox(self) -> tuple:
        los, his = zip(*(p.bbox() for p in self.pieces))
        return (tuple(min(v[i] for v in los) for i in range(self.s)),
                tuple(max(v[i] for v in his) for i in range(self.s)))

    def validate(self, lattice=None, samples: int = 8, rng_seed: int = 7) -> None:
        """Structural checks that need no polytope volumes (see the module docstring);
        raises SplineError.  `lattice` (a lattice.IntegerLattice) enables the exact
        partition-of-unity check at `samples` random rational points."""
        if not self.pieces:
            raise SplineError("no pieces")
        for i, p in enumerate(self.pieces):
            if p.poly.degree() > self.degree_bound:
                raise SplineError(f"piece {i} exceeds the declared degree bound")
            p.vertices()
        rng = random.Random(rng_seed)
        for i, p in enumerate(self.pieces):
            vs = p.vertices()
            w = [Fraction(rng.randint(1, 64)) for _ in vs]
            tot = sum(w)
            x = [sum(wi * v[k] for wi, v in zip(w, vs)) / tot for k in range(self.s)]
            if p.poly.eval(x) < 0:
                raise SplineError(f"spline is negative inside piece {i}")
        if lattice is not None:
            from .lattice import decompose_cartesian

            sol = SplineOnLattice(self, lattice, decompose_cartesian(lattice))
            pts = [tuple(Fraction(rng.randint(-128, 128), 97) for _ in range(self.s)) for _ in range(samples)]
            sol.check_partition_of_unity(pts)

    def __repr__(self) -> str:
        return f"PiecewisePolySpline({self.name or 'anon'}, s={self.s}, pieces={len(self.pieces)})"


def format_pp_spline(spline: PiecewisePolySpline) -> str:
    """The reference's document text (spline.py:645-664)."""
    out = [f"{MAGIC} {VERSION}", f"dim {spline.s}", f"degree {spline.degree_bound}"]
    if spline.name:
        out.append(f"name {spline.name}")
    if spline.center is not None:
        out.append("center " + " ".join(frac_str(c) for c in spline.center))
    for p in spline.pieces:
        out.append("piece")
        out.extend("hs " + " ".join(str(int(v)) for v in n) + " " + frac_str(o) for n, o in p.halfspaces)
        out.append("poly")
        out.extend("term " + " ".join(str(e) for e in exps) + " " + frac_str(p.poly.terms[exps])
                   for exps in sorted(p.poly.terms))
        out.append("end")
    return "\n".join(out) + "\n"


def import_pp_spline(text: str, validate: bool = True, lattice=None) -> PiecewisePolySpline:
    """Parse a `.spp` document (spline.py:667-743); malformed documents raise SplineError."""
    lines = [ln.strip() for ln in text.splitlines() if ln.strip() and not ln.startswith("#")]
    if not lines or not lines[0].startswith(MAGIC):
        raise SplineError("not a spline description document")
    head = lines[0].split()
    if (head[1] if len(head) > 1 else "?") != VERSION:
        raise SplineError("unsupported format version")
    dim = degree = None
    name, center, pieces = "", None, []
    i = 1
    while i < len(lines):
        parts = lines[i].split()
        key = parts[0]
        if key == "dim":
            dim = int(parts[1])
        elif key == "degree":
            degree = int(parts[1])
        elif key == "name":
            name = parts[1]
        elif key == "center":
            center = tuple(frac(t) for t in parts[1:])
        elif key == "piece":
            if dim is None or degree is None:
                raise SplineError("piece before dim/degree header")
            hs, terms, mode = [], {}, "hs"
            i += 1
            while True:
                if i >= len(lines):
                    raise SplineError("unterminated piece record")
                parts = lines[i].split()
                if parts[0] == "hs":
                    if len(parts) != dim + 2:
                        raise SplineError(f"bad half-space line: {lines[i]}")
                    hs.append((tuple(int(v) for v in parts[1:dim + 1]), frac(parts[dim + 1])))
                elif parts[0] == "poly":
                    mode = "poly"
                elif parts[0] == "term":
                    if mode != "poly" or len(parts) != dim + 2:
                        raise SplineError(f"bad term line: {lines[i]}")
                    terms[tuple(int(v) for v in parts[1:dim + 1])] = frac(parts[dim + 1])
                elif parts[0] == "end":
                    if not hs:
                        raise SplineError("piece without half-spaces")
                    pieces.append(SplinePiece(hs, Poly(dim, terms)))
                    break
                else:
                    raise SplineError(f"unexpected line in piece: {lines[i]}")
                i += 1
        else:
            raise SplineError(f"unexpected line: {lines[i]}")
        i += 1
    if dim is None or degree is None or not pieces:
        raise SplineError("incomplete spline description")
    sp = PiecewisePolySpline(dim, pieces, degree, name=name, center=center)
    for p in pieces:
        if p.poly.degree() > degree:
            raise SplineError("piece polynomial exceeds the declared degree bound")
    if validate:
        sp.validate(lattice=lattice)
    return sp


class SplineOnLattice:
    """spline.py:576-637: the spline paired with its lattice; weights carry |det L| so
    that shifts over the lattice form a partition of unity."""

    def __init__(self, spline: PiecewisePolySpline, lat, cosets):
        if spline.s != lat.s:
            raise SplineError("spline/lattice dimension mismatch")
        self.spline = spline
        self.lattice = lat
        self.cosets = cosets
        self.scale = Fraction(lat.det())

    def weight_eval(self, x: Sequence) -> Fraction:
        return self.scale * self.spline.eval_exact(x)

    def weight_poly(self, piece_index: int) -> Poly:
        p = self.spline.pieces[piece_index].poly
        return Poly(p.dim, {e: c * self.scale for e, c in p.terms.items()})

    def contributing_sites(self, x: Sequence) -> list:
        """Lattice sites m with x - m in the support (lexicographic order)."""
        x = [Fraction(v) for v in x]
        lo, hi = self.spline.support_bbox()
        rng = [range(-floor(-(xi - h)), floor(xi - l) + 1) for xi, l, h in zip(x, lo, hi)]
        out = []
        for m in product(*rng):
            if self.lattice.contains_site(m):
                d = [xi - mi for xi, mi in zip(x, m)]
                if self.spline.piece_at(d) is not None:
                    out.append(tuple(int(v) for v in m))
        return out

    def partition_of_unity_at(self, x: Sequence) -> Fraction:
        x = [Fraction(v) for v in x]
        return sum((self.weight_eval([xi - mi for xi, mi in zip(x, m)]) for m in self.contributing_sites(x)),
                   Fraction(0))

    def check_partition_of_unity(self, points) -> None:
        for x in points:
            tot = self.partition_of_unity_at(x)
            if tot != 1:
                raise SplineError(f"partition of unity fails at {tuple(x)}: sum {tot}")
