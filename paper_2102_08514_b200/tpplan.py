"""Native plan producer for tensor-product B-splines (TP family).

The reference builds a tensor-product plan (E3 x (n+1) on CC3, e.g. cc_tricubic) by exact
PP extraction of the box spline (spline.py:481-531), sub-region analysis and symmetry search
(analysis.py:113-399) and plan assembly (plancompile.py:328-380): 75 s + 28 s of exact host
arithmetic for the tricubic.  For this family every step has a closed form, so the plan is
produced here directly (seconds instead of minutes) for any degree:

* one sub-region per unit cell: no cut planes (Q = 0), r = 1, sigma = [0], one class with the
  identity transform (analysis.py:89-100 with T = I, t = 0, pi = identity);
* the kernel's sites are the offsets [-n, 0]^3 in sorted order (analysis.py:236-237), each
  weighted by the product of the 1-D cardinal B-spline pieces in y = x - floor(x)
  (exact.tensor_site_weight, Cox-de Boor in rationals);
* fetch grouping = the reference's rule (plancompile.py:150-246): candidate groups are the
  axis-aligned pairs / squares / cubes of sites whose weight tensor factors rank-1 (checked
  as exact polynomial identities), the cover is an exact cover of minimum cardinality with
  ties broken toward the lexicographically smallest list of sorted site-index tuples, and
  groups are listed by (-size, sites);
* fetch ordering = the reference's cost model (plancompile.py:271-325): new texels per fetch
  of each group's hardware-fetch footprint, exhaustive over permutations for <= 8 groups,
  nearest-neighbour otherwise.

The result is the same EvaluationPlan the reference compiler emits — same canonical JSON,
same checksum — which tests/test_tpplan.py checks against reference-compiled plans
(degrees 1 and 3 from the catalog, 2 and 4 from tests/golden/tp_plans/).
"""

from __future__ import annotations

from fractions import Fraction
from math import gcd
from itertools import combinations, permutations, product
from typing import Sequence

from .exact import Poly, tensor_site_weight
from .plan import ClassTransform, EvaluationPlan, FetchGroup, PlanError, PlanKernel, PlanOptions


def _rank1_group(corners: list, axes: tuple, weight_of: dict):
    """FetchGroup of `corners` (tensor-corner order over `axes`) when the corner weights
    factor as g * prod_j (t_j | 1 - t_j), else None (plancompile.py:207-232)."""
    ws = [weight_of[c] for c in corners]
    g = ws[0]
    for w in ws[1:]:
        g = g + w
    if g.is_zero():
        return None
    k = len(axes)
    t_nums = []
    for j in range(k):
        t = Poly(g.dim)
        for idx, w in enumerate(ws):
            if idx >> j & 1:
                t = t + w
        t_nums.append(t)
    if k > 1:
        one = Poly.const(g.dim, 1)
        for idx, w in enumerate(ws):
            lhs = w
            for _ in range(k - 1):
                lhs = lhs * g
            rhs = one
            for j in range(k):
                rhs = rhs * (t_nums[j] if idx >> j & 1 else g - t_nums[j])
            if lhs != rhs:
                return None
    return FetchGroup(tuple(corners), tuple(axes), g, tuple(t_nums))


def _min_exact_cover(n: int, rows: list) -> list:
    """Smallest exact cover of {0..n-1} by `rows` (sets of indices); among the smallest, the
    one whose sorted list of sorted index tuples is least — the cover the reference's
    exhaustive search returns (plancompile.py:233-268), found without enumerating every
    minimum cover:

    * the minimum cardinality k comes from a feasibility search ("coverable with <= m rows?")
      pruned by the fractional bound sum_e 1/maxrow(e) (each chosen row contributes <= 1),
      with failed (set, m) states memoised;
    * the least key is then built greedily: in any exact cover the row holding the smallest
      uncovered element sorts first among the rows still to choose, so taking, for that
      element, the least row tuple that still admits a cover of the remaining budget is
      lexicographically optimal.
    """
    masks = [sum(1 << e for e in row) for row in rows]
    sizes = [len(r) for r in rows]
    by_elem = [[] for _ in range(n)]
    for i, row in enumerate(rows):
        for e in row:
            by_elem[e].append(i)
    unit = 1
    for sz in set(sizes):
        unit = unit * sz // gcd(unit, sz)
    wt = [unit // max((sizes[i] for i in by_elem[e]), default=1) for e in range(n)]
    fail: dict = {}

    def bound(left: int) -> int:
        tot, m = 0, left
        while m:
            low = m & -m
            tot += wt[low.bit_length() - 1]
            m ^= low
        return -(-tot // unit)

    def usable(e: int, left: int) -> list:
        return [i for i in by_elem[e] if masks[i] & ~left == 0]

    def feasible(left: int, m: int) -> bool:
        if not left:
            return True
        if m <= 0 or bound(left) > m or fail.get(left, -1) >= m:
            return False
        e_best, use_best, mm = -1, None, left
        while mm:
            low = mm & -mm
            e = low.bit_length() - 1
            mm ^= low
            use = usable(e, left)
            if use_best is None or len(use) < len(use_best):
                e_best, use_best = e, use
                if len(use) <= 1:
                    break
        for i in sorted(use_best, key=lambda i: -sizes[i]):
            if feasible(left & ~masks[i], m - 1):
                return True
        fail[left] = max(fail.get(left, -1), m)
        return False

    full = (1 << n) - 1
    k = bound(full)
    while not feasible(full, k):
        k += 1
    chosen, left = [], full
    while left:
        e = (left & -left).bit_length() - 1
        for i in sorted(usable(e, left), key=lambda i: tuple(sorted(rows[i]))):
            if feasible(left & ~masks[i], k - len(chosen) - 1):
                chosen.append(i)
                left &= ~masks[i]
                break
        else:  # pragma: no cover - feasible(full, k) guarantees a continuation
            raise PlanError("no exact cover of the kernel sites")
    return chosen


def _cover_and_sort(sites: list, cands: list) -> tuple:
    index = {s: i for i, s in enumerate(sites)}
    rows = [frozenset(index[s] for s in g.sites) for g in cands]
    chosen = _min_exact_cover(len(sites), rows)
    return tuple(sorted((cands[i] for i in chosen), key=lambda g: (-g.size, g.sites)))


def group_fetches(sites: Sequence[tuple], weights: Sequence[Poly], diag: Sequence[int], grouped: bool = True,
                  max_group_dim: int = 3) -> tuple:
    """plancompile.py:150-204 semantics: minimum exact cover by rank-1 groups."""
    sites = [tuple(s) for s in sites]
    weight_of = dict(zip(sites, weights))
    singles = [FetchGroup((s,), (), weight_of[s], ()) for s in sites]
    if not grouped:
        return tuple(singles)
    dim = len(diag)
    cands = list(singles)
    for k in range(1, min(max_group_dim, dim) + 1):
        for axes in combinations(range(dim), k):
            for base in sites:
                corners = []
                for idx in range(1 << k):
                    c = list(base)
                    for j in range(k):
                        if idx >> j & 1:
                            c[axes[j]] += diag[axes[j]]
                    c = tuple(c)
                    if c not in weight_of:
                        break
                    corners.append(c)
                else:
                    grp = _rank1_group(corners, axes, weight_of)
                    if grp is not None:
                        cands.append(grp)
    return _cover_and_sort(sites, cands)


def _tp_cover(degree: int, sites: list, cands: list) -> tuple:
    """The cover group_fetches picks, found directly for tensor-product kernels.

    Lower bound: sites whose offsets o + n are all even are pairwise separated by >= 2 along
    some axis, and a group spans <= 2 consecutive offsets per axis, so no group holds two of
    them: every cover has >= ceil((n+1)/2)^3 groups (and >= sites / 8), and the per-axis
    product of pairs (plus one single when n+1 is odd) attains it.  Among covers of that size the reference keeps
    the least sorted list of sorted site-index tuples (plancompile.py:234-262); groups are
    disjoint and each holds its smallest index, so that list is the chosen groups ordered
    by their smallest index — a depth-first search that always extends the smallest
    uncovered index with its candidate groups in increasing tuple order, pruned by the
    bound, meets the answer first."""
    index = {s: i for i, s in enumerate(sites)}
    rows = [tuple(sorted(index[s] for s in g.sites)) for g in cands]
    masks = [sum(1 << e for e in r) for r in rows]
    indep = 0
    for s, i in index.items():
        if all((o + degree) % 2 == 0 for o in s):
            indep |= 1 << i
    target = bin(indep).count("1")
    by_first = {}
    for ci, r in enumerate(rows):
        by_first.setdefault(r[0], []).append(ci)
    for lst in by_first.values():
        lst.sort(key=lambda ci: rows[ci])
    chosen = []

    def search(left: int) -> bool:
        if not left:
            return True
        e = (left & -left).bit_length() - 1
        for ci in by_first.get(e, ()):
            m = masks[ci]
            if m & ~left:
                continue
            rest = left & ~m
            need = max(bin(rest & indep).count("1"), -(-bin(rest).count("1") // 8))  # both bounds
            if len(chosen) + 1 + need > target:
                continue
            chosen.append(ci)
            if search(rest):
                return True
            chosen.pop()
        return False

    if not search((1 << len(sites)) - 1):
        raise PlanError("no minimum cover of the tensor-product sites")
    return tuple(sorted((cands[i] for i in chosen), key=lambda g: (-g.size, g.sites)))


def _tp_candidates(degree: int, sites: list) -> list:
    """group_fetches' candidate list for tensor-product weights, in the same order (singles,
    then pairs / squares / cubes by axis set and base site), built from the 1-D pieces: the
    weight of site o is prod_i p_{o_i}(y_i), so every axis-aligned box of sites factors rank-1
    with g = prod_{i spanned} (p_{b_i} + p_{b_i + 1}) prod_{i not spanned} p_{b_i} and t_num_j
    = g with axis j's factor replaced by p_{b_j + 1} (the identities _rank1_group checks)."""
    from .exact import bspline_piece_polys

    dim = 3
    pieces = bspline_piece_polys(degree)

    def p1(axis: int, off: int) -> Poly:
        e = [0] * dim
        terms = {}
        for k, c in enumerate(pieces[off + degree]):
            e[axis] = k
            terms[tuple(e)] = c
        return Poly(dim, terms)

    one = Poly.const(dim, 1)
    weight = {}
    for s in sites:
        w = one
        for i in range(dim):
            w = w * p1(i, s[i])
        weight[s] = w
    cands = [FetchGroup((s,), (), weight[s], ()) for s in sites]
    siteset = set(sites)
    for k in range(1, dim + 1):
        for axes in combinations(range(dim), k):
            for base in sites:
                corners = []
                for idx in range(1 << k):
                    c = list(base)
                    for j in range(k):
                        if idx >> j & 1:
                            c[axes[j]] += 1
                    corners.append(tuple(c))
                if not all(c in siteset for c in corners):
                    continue
                fac = [p1(i, base[i]) + p1(i, base[i] + 1) if i in axes else p1(i, base[i]) for i in range(dim)]
                g = fac[0] * fac[1] * fac[2]
                t_nums = []
                for a in axes:
                    f = list(fac)
                    f[a] = p1(a, base[a] + 1)
                    t_nums.append(f[0] * f[1] * f[2])
                cands.append(FetchGroup(tuple(corners), tuple(axes), g, tuple(t_nums)))
    return cands


def _footprint(group: FetchGroup, diag: Sequence[int], hi: Sequence[int]) -> frozenset:
    """Texels one hardware linear fetch of `group` touches (plancompile.py:271-291):
    spanned axes its two texel planes, other axes the neighbour toward the interior."""
    lo = [min(s[i] // diag[i] for s in group.sites) for i in range(len(diag))]
    spans = []
    for i in range(len(diag)):
        if i in group.span_axes or lo[i] < hi[i]:
            spans.append((lo[i], lo[i] + 1))
        else:
            spans.append((lo[i] - 1, lo[i]))
    return frozenset(product(*[range(a, b + 1) for a, b in spans]))


def _order_cost(feet) -> int:
    cost, prev = 0, frozenset()
    for f in feet:
        cost += len(f - prev)
        prev = f
    return cost


def order_fetches(groups: Sequence[FetchGroup], diag: Sequence[int]) -> tuple:
    """plancompile.py:294-325 semantics: minimise new texels per fetch; exhaustive for <= 8
    groups (first minimum in permutation order), nearest-neighbour from the first otherwise."""
    groups = list(groups)
    if len(groups) <= 1:
        return tuple(groups)
    dim = len(diag)
    zs = [tuple(s[i] // diag[i] for i in range(dim)) for g in groups for s in g.sites]
    hi = tuple(max(z[i] for z in zs) for i in range(dim))
    feet = [_footprint(g, diag, hi) for g in groups]
    if len(groups) <= 8:
        best, best_cost = None, None
        for perm in permutations(range(len(groups))):
            c = _order_cost([feet[i] for i in perm])
            if best_cost is None or c < best_cost:
                best, best_cost = perm, c
        return tuple(groups[i] for i in best)
    left = list(range(len(groups)))
    seq = [left.pop(0)]
    while left:
        prev = feet[seq[-1]]
        nxt = min(left, key=lambda i: (len(feet[i] - prev), i))
        left.remove(nxt)
        seq.append(nxt)
    return tuple(groups[i] for i in seq)


def tensor_product_plan(degree: int, name: str | None = None, options: PlanOptions | None = None) -> EvaluationPlan:
    """EvaluationPlan of the degree-n tensor-product B-spline (E3 x (n+1)) on CC3, as the
    reference compiler would emit it (module docstring)."""
    if degree < 0:
        raise PlanError("degree must be >= 0")
    options = options or PlanOptions()
    s = 3
    sites = sorted(product(range(-degree, 1), repeat=s))
    diag = (1, 1, 1)
    if options.grouped:
        groups = _tp_cover(degree, sites, _tp_candidates(degree, sites))
    else:
        groups = tuple(FetchGroup((site,), (), tensor_site_weight(degree, s, site), ()) for site in sites)
    if options.ordered:
        groups = order_fetches(groups, diag)
    one, zero = Fraction(1), Fraction(0)
    ident = tuple(tuple(one if i == j else zero for j in range(s)) for i in range(s))
    cls = ClassTransform(kernel=0, T=ident, t=(zero,) * s,
                         pi_linear=tuple(tuple(int(i == j) for j in range(s)) for i in range(s)), pi_offset=(0,) * s)
    return EvaluationPlan(
        name=name or f"cc_tp{degree}",
        lattice_name="CC3",
        s=s,
        diag=diag,
        shifts=((0, 0, 0),),
        scale=Fraction(1),
        planes=(),
        r=1,
        sigma=(0,),
        classes=(cls,),
        kernels=(PlanKernel(0, tuple(groups)),),
        options=options,
        basis_nonnegative=True,
        pou_on_sublattice=True,
        reflective_axes=(True,) * s,
    )
