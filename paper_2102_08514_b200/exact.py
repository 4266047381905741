"""Exact rational polynomials: just enough for plan loading and plan specialisation.

The reference computes everything before the hot path in exact rationals
(`exactmath.py:1-587`).  The hot path itself only needs a plan's weight
polynomials (`FetchGroup.g` / `t_nums`, plancompile.py:55-77), so this module keeps a
small `Poly` (exponent tuple -> Fraction) with the operations the host side uses:

* parsing the plan wire format (`plancompile.py:402-407`),
* exact identities, e.g. proving that a plan is a tensor-product B-spline before
  routing it to the separable kernel (see `tensor_bspline_degree`),
* a greedy Horner factorisation for the code generator.  The pivot rule is the one
  the reference documents for `horner_factor` (`exactmath.py:543-587`: variable in
  the most remaining terms, ties toward the lowest index), re-implemented here as
  an expression tree instead of an SSA op list.
"""

from __future__ import annotations

from fractions import Fraction
from itertools import product
from typing import Dict, Iterable, Sequence, Tuple

Exps = Tuple[int, ...]


def frac(text) -> Fraction:
    """Parse 'num' or 'num/den' (the plan wire format, plancompile.py:402-407)."""
    if isinstance(text, Fraction):
        return text
    if isinstance(text, int):
        return Fraction(text)
    return Fraction(str(text).strip())


def frac_str(q: Fraction) -> str:
    q = Fraction(q)
    return str(q.numerator) if q.denominator == 1 else f"{q.numerator}/{q.denominator}"


class Poly:
    """Multivariate polynomial with rational coefficients; zero terms are never stored."""

    __slots__ = ("dim", "terms")

    def __init__(self, dim: int, terms: Dict[Exps, Fraction] | None = None):
        self.dim = dim
        self.terms: Dict[Exps, Fraction] = {}
        for e, c in (terms or {}).items():
            c = Fraction(c)
            if c != 0:
                if len(e) != dim:
                    raise ValueError("exponent length does not match the dimension")
                self.terms[tuple(int(v) for v in e)] = c

    # -- constructors --------------------------------------------------------
    @staticmethod
    def const(dim: int, c) -> "Poly":
        return Poly(dim, {(0,) * dim: Fraction(c)})

    @staticmethod
    def var(dim: int, i: int) -> "Poly":
        e = [0] * dim
        e[i] = 1
        return Poly(dim, {tuple(e): Fraction(1)})

    @staticmethod
    def from_obj(dim: int, obj: Iterable) -> "Poly":
        return Poly(dim, {tuple(e): frac(c) for e, c in obj})

    def to_obj(self) -> list:
        return [[list(e), frac_str(c)] for e, c in sorted(self.terms.items())]

    # -- algebra ---------------------------------------------------------------
    def is_zero(self) -> bool:
        return not self.terms

    def degree(self) -> int:
        return max((sum(e) for e in self.terms), default=0)

    def __add__(self, other: "Poly") -> "Poly":
        out = dict(self.terms)
        for e, c in other.terms.items():
            out[e] = out.get(e, Fraction(0)) + c
        return Poly(self.dim, out)

    def __neg__(self) -> "Poly":
        return Poly(self.dim, {e: -c for e, c in self.terms.items()})

    def __sub__(self, other: "Poly") -> "Poly":
        return self + (-other)

    def __mul__(self, other: "Poly") -> "Poly":
        out: Dict[Exps, Fraction] = {}
        for e1, c1 in self.terms.items():
            for e2, c2 in other.terms.items():
                e = tuple(a + b for a, b in zip(e1, e2))
                out[e] = out.get(e, Fraction(0)) + c1 * c2
        return Poly(self.dim, out)

    def divexact(self, d: "Poly") -> "Poly":
        """Exact quotient self / d (multivariate division in lex order); raises ValueError
        when d does not divide self."""
        if d.is_zero():
            raise ZeroDivisionError("division by the zero polynomial")
        lead_d = max(d.terms)
        cd = d.terms[lead_d]
        rem = Poly(self.dim, self.terms)
        quo: Dict[Exps, Fraction] = {}
        while not rem.is_zero():
            lead = max(rem.terms)
            if any(a < b for a, b in zip(lead, lead_d)):
                raise ValueError("polynomial division is not exact")
            e = tuple(a - b for a, b in zip(lead, lead_d))
            c = rem.terms[lead] / cd
            quo[e] = quo.get(e, Fraction(0)) + c
            rem = rem - Poly(self.dim, {e: c}) * d
        return Poly(self.dim, quo)

    def __eq__(self, other) -> bool:
        return isinstance(other, Poly) and self.dim == other.dim and self.terms == other.terms

    def __hash__(self) -> int:
        return hash((self.dim, frozenset(self.terms.items())))

    def __repr__(self) -> str:
        return f"Poly({self.dim}, {self.to_obj()})"

    def eval(self, point: Sequence) -> Fraction:
        pt = [Fraction(p) for p in point]
        acc = Fraction(0)
        for e, c in self.terms.items():
            m = c
            for v, k in zip(pt, e):
                if k:
                    m *= v ** k
            acc += m
        return acc

    def eval_float(self, point: Sequence[float]) -> float:
        acc = 0.0
        for e, c in self.terms.items():
            m = float(c)
            for v, k in zip(point, e):
                if k:
                    m *= float(v) ** k
            acc += m
        return acc


# ---------------------------------------------------------------------------
# Horner expression trees for the code generator


class HNode:
    """Expression node: ('const', q) | ('var', i) | ('add', a, b) | ('mul', a, b) | ('fma', a, b, c)."""

    __slots__ = ("kind", "args")

    def __init__(self, kind: str, *args):
        self.kind = kind
        self.args = args

    def mul_count(self) -> int:
        own = 1 if self.kind in ("mul", "fma") else 0
        return own + sum(a.mul_count() for a in self.args if isinstance(a, HNode))


def horner_tree(p: Poly) -> HNode:
    """Greedy multivariate Horner form of p (pivot: most terms, ties: lowest index)."""
    if p.is_zero():
        return HNode("const", Fraction(0))
    if all(sum(e) == 0 for e in p.terms):
        return HNode("const", next(iter(p.terms.values())))
    counts = [0] * p.dim
    for e in p.terms:
        for i, k in enumerate(e):
            if k:
                counts[i] += 1
    pivot = max(range(p.dim), key=lambda i: (counts[i], -i))
    q: Dict[Exps, Fraction] = {}
    r: Dict[Exps, Fraction] = {}
    for e, c in p.terms.items():
        if e[pivot]:
            red = list(e)
            red[pivot] -= 1
            q[tuple(red)] = c
        else:
            r[e] = c
    qp = Poly(p.dim, q)
    rp = Poly(p.dim, r)
    x = HNode("var", pivot)
    one = (0,) * p.dim
    q_is_one = qp.terms == {one: Fraction(1)}
    qn = None if q_is_one else horner_tree(qp)
    if rp.is_zero():
        return x if q_is_one else HNode("mul", x, qn)
    rn = horner_tree(rp)
    if q_is_one:
        return HNode("add", x, rn)
    return HNode("fma", x, qn, rn)


# ---------------------------------------------------------------------------
# Uniform B-splines (non-centred, support [0, n+1]) for tensor-product detection


def bspline_piece_polys(degree: int) -> list:
    """1-D cardinal B-spline of the given degree on [0, degree+1], as polynomials in
    the local offset t in [0,1): entry a is the weight of site  floor(x) - degree + a.

    Non-centred convention of the reference: a box spline's support is the Minkowski
    sum of [0, xi_i] (polytope.py:346-400), so E3 x (degree+1) has support [0, degree+1]^3.
    """
    # Piece j of the B-spline on [j, j+1) as a polynomial in u, via the Cox-de Boor
    # recursion on integer knots, done exactly.
    pieces = [[Fraction(1)]]  # degree 0: 1 on [0,1)
    for n in range(1, degree + 1):
        # N_n(u) = u/n N_{n-1}(u) + (n+1-u)/n N_{n-1}(u-1)
        new = []
        for j in range(n + 1):
            acc = [Fraction(0)] * (n + 1)
            if j < n:  # u/n * N_{n-1} piece j  (in u)
                for k, c in enumerate(pieces[j]):
                    acc[k + 1] += c / n
            if j >= 1:  # (n+1-u)/n * N_{n-1}(u-1) piece j-1 shifted by 1
                shifted = _shift_poly(pieces[j - 1], -1)
                for k, c in enumerate(shifted):
                    acc[k] += c * (n + 1) / n
                    acc[k + 1] -= c / n
            new.append(acc)
        pieces = new
    # site n = i - degree + a with x = i + t  ->  u = x - n = t + degree - a, piece index degree - a
    out = []
    for a in range(degree + 1):
        j = degree - a
        out.append(_shift_poly(pieces[j], j))  # substitute u = t + j
    return out


def _shift_poly(coeffs: Sequence[Fraction], h) -> list:
    """Coefficients (in t) of p(t + h) for p given by ascending coefficients."""
    from math import comb

    n = len(coeffs)
    out = [Fraction(0)] * n
    for k, c in enumerate(coeffs):
        for i in range(k + 1):
            out[i] += c * comb(k, i) * Fraction(h) ** (k - i)
    return out


def tensor_site_weight(degree: int, dim: int, offsets: Sequence[int]) -> Poly:
    """Weight polynomial, in y = x - floor(x) in [0,1)^dim, of the site floor(x) + offsets."""
    pieces = bspline_piece_polys(degree)
    poly = Poly.const(dim, 1)
    for axis, off in enumerate(offsets):
        a = off + degree
        if not 0 <= a <= degree:
            return Poly(dim)
        coeffs = pieces[a]
        terms = {}
        for k, c in enumerate(coeffs):
            e = [0] * dim
            e[axis] = k
            terms[tuple(e)] = c
        poly = poly * Poly(dim, terms)
    return poly


def all_offsets(degree: int, dim: int):
    return product(range(-degree, 1), repeat=dim)
