"""Evaluation plans: the hot path's input data contract and its JSON wire format.

Mirrors the reference data model (`plancompile.py:47-143`, `analysis.py:89-100`):
`PlanOptions`, `FetchGroup`, `PlanKernel`, `ClassTransform`, `EvaluationPlan`, and the
checksummed JSON document of `serialize_plan` / `deserialize_plan`
(`plancompile.py:418-557`).  Plans are produced by the reference compiler (the
compile passes are out of scope); this module loads, validates and
*specialises* them for the B200 kernels:

* `ClassTransform` matrices are reduced to signed permutations (probe12, SURVEY.md §9:
  every corpus T is a signed permutation with integral t and piA = T^-1);
* the per-coset site reach (halo) is derived from the mapped sites;
* `tensor_bspline_degree` proves, by exact polynomial identities, that a plan is the
  separable tensor-product B-spline of some degree so it can use the separable kernel.
"""

from __future__ import annotations

import hashlib
import json
from dataclasses import dataclass, field
from fractions import Fraction
from typing import Optional, Sequence, Tuple

from .exact import Poly, all_offsets, frac, frac_str, tensor_site_weight

SIGMA_SENTINEL = -1  # analysis.py:39

_PLAN_FORMAT = "splineplan-plan"  # plancompile.py:398-399
_PLAN_VERSION = 1


class PlanError(ValueError):
    """Malformed or unsupported plan (reference: plancompile.py:43-44)."""


@dataclass(frozen=True)
class PlanOptions:
    """plancompile.py:47-52.  Only `texel_offset_half` touches evaluation in the
    reference (plancompile.py:696-697); the software local lerp used here is
    independent of it ('linear-fetch merge')."""

    grouped: bool = True
    predicated: bool = True
    ordered: bool = True
    texel_offset_half: bool = True


@dataclass(frozen=True)
class FetchGroup:
    """1, 2, 4 or 8 zero-coset sites served by one (multi)linear read (plancompile.py:55-77).

    Sites are in tensor-corner order over `span_axes` (bit j of the corner index steps
    along span_axes[j]); `g` is the weight sum and t_nums[j]/g the lerp parameter.
    """

    sites: tuple
    span_axes: tuple
    g: Poly
    t_nums: tuple

    @property
    def size(self) -> int:
        return len(self.sites)


@dataclass(frozen=True)
class PlanKernel:
    ref_class: int
    groups: tuple

    @property
    def nearest_count(self) -> int:
        return sum(g.size for g in self.groups)

    @property
    def grouped_count(self) -> int:
        return len(self.groups)


@dataclass(frozen=True)
class ClassTransform:
    """analysis.py:89-100: y = T x - t selects the reference kernel; sites map by pi."""

    kernel: int
    T: tuple          # s x s rationals
    t: tuple          # s rationals
    pi_linear: tuple  # s x s ints
    pi_offset: tuple  # s ints

    def map_site(self, site: Sequence[int]) -> tuple:
        return tuple(
            sum(int(a) * int(v) for a, v in zip(row, site)) + int(o)
            for row, o in zip(self.pi_linear, self.pi_offset)
        )


@dataclass
class EvaluationPlan:
    """plancompile.py:94-143."""

    name: str
    lattice_name: str
    s: int
    diag: tuple
    shifts: tuple
    scale: Fraction
    planes: tuple       # ((normal ints), Fraction offset)
    r: int
    sigma: tuple
    classes: tuple
    kernels: tuple
    options: PlanOptions
    basis_nonnegative: bool
    pou_on_sublattice: bool
    reflective_axes: tuple
    octant_fold: bool = False
    checksum: str = field(default="", compare=False)

    @property
    def M(self) -> int:
        return len(self.shifts)

    @property
    def N(self) -> int:
        return len(self.classes)

    @property
    def Q(self) -> int:
        return len(self.planes)

    @property
    def K(self) -> int:
        return len(self.kernels)

    def nearest_fetch_counts(self) -> tuple:
        """plancompile.py:129-134."""
        return tuple(self.M * self.kernels[c.kernel].nearest_count for c in self.classes)

    def grouped_fetch_counts(self) -> tuple:
        """plancompile.py:136-140."""
        return tuple(self.M * self.kernels[c.kernel].grouped_count for c in self.classes)

    def __eq__(self, other) -> bool:
        return isinstance(other, EvaluationPlan) and plan_to_dict(self) == plan_to_dict(other)

    # -- specialisation helpers (B200 side) ------------------------------------

    def site_reach(self) -> Tuple[tuple, tuple]:
        """Per-axis [lo, hi] of coset cell offsets any class may read, relative to the
        point's cell floor((x - l_k)/d).  Mapped sites piA*site + pib are multiples of d
        (probe11), so the offsets are integers."""
        lo = [0] * self.s
        hi = [0] * self.s
        first = True
        for ct in self.classes:
            for g in self.kernels[ct.kernel].groups:
                for site in g.sites:
                    m = ct.map_site(site)
                    for i in range(self.s):
                        if m[i] % self.diag[i]:
                            raise PlanError("mapped site is not on the zero coset")
                        z = m[i] // self.diag[i]
                        if first:
                            lo[i] = hi[i] = z
                        else:
                            lo[i] = min(lo[i], z)
                            hi[i] = max(hi[i], z)
                    first = False
        return tuple(lo), tuple(hi)

    def signed_permutation_classes(self) -> Optional[list]:
        """Per class (kernel, perm, sign, t, rho, tau, pib) when every T and piA is a
        signed permutation and t is integral; None otherwise (general path)."""
        out = []
        for ct in self.classes:
            T = [[Fraction(v) for v in row] for row in ct.T]
            sp = _signed_perm(T)
            A = [[Fraction(int(v)) for v in row] for row in ct.pi_linear]
            sa = _signed_perm(A)
            if sp is None or sa is None:
                return None
            if any(Fraction(v).denominator != 1 for v in ct.t):
                return None
            perm, sign = sp
            rho, tau = sa
            out.append(
                dict(
                    kernel=ct.kernel,
                    perm=perm,
                    sign=sign,
                    t=tuple(int(Fraction(v)) for v in ct.t),
                    rho=rho,
                    tau=tau,
                    pib=tuple(int(v) for v in ct.pi_offset),
                )
            )
        return out

    def tensor_bspline_degree(self) -> Optional[int]:
        """Degree n if this plan evaluates  sum_m c_m prod_i B_n(x_i - m_i)  exactly
        (B_n the non-centred cardinal B-spline on [0, n+1]); None otherwise.

        Proof obligation, all in exact rationals: Cartesian lattice, one coset, one class
        with the identity transform, and for every fetch group the reconstructed corner
        weights  g * prod_j (t_j/g | 1 - t_j/g)  equal the tensor-product weights:
        w_site * g^(k-1) == prod_j (t_num_j | g - t_num_j)  (plancompile.py:218-229).
        """
        if self.M != 1 or any(d != 1 for d in self.diag) or self.Q != 0 or self.N != 1 or self.K != 1:
            return None
        ct = self.classes[0]
        ident = tuple(tuple(Fraction(int(i == j)) for j in range(self.s)) for i in range(self.s))
        if tuple(tuple(Fraction(v) for v in row) for row in ct.T) != ident:
            return None
        if any(Fraction(v) != 0 for v in ct.t) or any(int(v) != 0 for v in ct.pi_offset):
            return None
        if tuple(tuple(int(v) for v in row) for row in ct.pi_linear) != tuple(
            tuple(int(i == j) for j in range(self.s)) for i in range(self.s)
        ):
            return None
        sites = [tuple(site) for g in self.kernels[0].groups for site in g.sites]
        if not sites:
            return None
        degree = -min(min(site) for site in sites)
        expected = {tuple(o) for o in all_offsets(degree, self.s)}
        if set(sites) != expected or len(sites) != len(expected):
            return None
        one = Poly.const(self.s, 1)
        for g in self.kernels[0].groups:
            k = len(g.span_axes)
            gk = one
            for _ in range(max(k - 1, 0)):
                gk = gk * g.g
            for idx, site in enumerate(g.sites):
                lhs = tensor_site_weight(degree, self.s, site) * gk
                rhs = one
                if k == 0:
                    rhs = g.g
                for j in range(k):
                    rhs = rhs * (g.t_nums[j] if (idx >> j) & 1 else g.g - g.t_nums[j])
                if lhs != rhs:
                    return None
        return degree


def _signed_perm(m) -> Optional[Tuple[tuple, tuple]]:
    """(perm, sign) with m[i][perm[i]] = sign[i] in {-1, 1} and zeros elsewhere."""
    s = len(m)
    perm = []
    sign = []
    for i in range(s):
        nz = [(j, v) for j, v in enumerate(m[i]) if v != 0]
        if len(nz) != 1 or abs(nz[0][1]) != 1:
            return None
        perm.append(nz[0][0])
        sign.append(int(nz[0][1]))
    if sorted(perm) != list(range(s)):
        return None
    return tuple(perm), tuple(sign)


# ---------------------------------------------------------------------------
# Wire format (plancompile.py:402-557)


def plan_to_dict(plan: EvaluationPlan) -> dict:
    return {
        "format": _PLAN_FORMAT,
        "version": _PLAN_VERSION,
        "header": {
            "name": plan.name,
            "lattice": plan.lattice_name,
            "s": plan.s,
            "diag": list(plan.diag),
            "shifts": [list(sh) for sh in plan.shifts],
            "scale": frac_str(plan.scale),
            "N": plan.N,
            "Q": plan.Q,
            "r": plan.r,
            "K": plan.K,
            "options": {
                "grouped": plan.options.grouped,
                "predicated": plan.options.predicated,
                "ordered": plan.options.ordered,
                "texel_offset_half": plan.options.texel_offset_half,
            },
            "basis_nonnegative": plan.basis_nonnegative,
            "pou_on_sublattice": plan.pou_on_sublattice,
            "reflective_axes": list(plan.reflective_axes),
            "octant_fold": plan.octant_fold,
        },
        "planes": [
            {"normal": list(n), "offset": frac_str(o), "offset_float": float(o)} for n, o in plan.planes
        ],
        "sigma": list(plan.sigma),
        "classes": [
            {
                "kernel": c.kernel,
                "T": [[frac_str(v) for v in row] for row in c.T],
                "t": [frac_str(v) for v in c.t],
                "T_float": [[float(v) for v in row] for row in c.T],
                "t_float": [float(v) for v in c.t],
                "piA": [[int(v) for v in row] for row in c.pi_linear],
                "pib": list(c.pi_offset),
            }
            for c in plan.classes
        ],
        "kernels": [
            {
                "ref_class": k.ref_class,
                "groups": [
                    {
                        "sites": [list(site) for site in g.sites],
                        "span_axes": list(g.span_axes),
                        "g": g.g.to_obj(),
                        "t_nums": [t.to_obj() for t in g.t_nums],
                    }
                    for g in k.groups
                ],
            }
            for k in plan.kernels
        ],
    }


def plan_from_dict(doc: dict) -> EvaluationPlan:
    try:
        hdr = doc["header"]
        s = int(hdr["s"])
        classes = tuple(
            ClassTransform(
                kernel=int(c["kernel"]),
                T=tuple(tuple(frac(v) for v in row) for row in c["T"]),
                t=tuple(frac(v) for v in c["t"]),
                pi_linear=tuple(tuple(int(v) for v in row) for row in c["piA"]),
                pi_offset=tuple(int(v) for v in c["pib"]),
            )
            for c in doc["classes"]
        )
        kernels = tuple(
            PlanKernel(
                ref_class=int(k["ref_class"]),
                groups=tuple(
                    FetchGroup(
                        sites=tuple(tuple(int(v) for v in site) for site in g["sites"]),
                        span_axes=tuple(int(a) for a in g["span_axes"]),
                        g=Poly.from_obj(s, g["g"]),
                        t_nums=tuple(Poly.from_obj(s, t) for t in g["t_nums"]),
                    )
                    for g in k["groups"]
                ),
            )
            for k in doc["kernels"]
        )
        opts = hdr["options"]
        plan = EvaluationPlan(
            name=hdr["name"],
            lattice_name=hdr["lattice"],
            s=s,
            diag=tuple(int(d) for d in hdr["diag"]),
            shifts=tuple(tuple(int(v) for v in sh) for sh in hdr["shifts"]),
            scale=frac(hdr["scale"]),
            planes=tuple((tuple(int(v) for v in p["normal"]), frac(p["offset"])) for p in doc["planes"]),
            r=int(hdr["r"]),
            sigma=tuple(int(v) for v in doc["sigma"]),
            classes=classes,
            kernels=kernels,
            options=PlanOptions(
                grouped=bool(opts["grouped"]),
                predicated=bool(opts["predicated"]),
                ordered=bool(opts["ordered"]),
                texel_offset_half=bool(opts["texel_offset_half"]),
            ),
            basis_nonnegative=bool(hdr["basis_nonnegative"]),
            pou_on_sublattice=bool(hdr["pou_on_sublattice"]),
            reflective_axes=tuple(bool(v) for v in hdr["reflective_axes"]),
            octant_fold=bool(hdr.get("octant_fold", False)),
        )
    except (KeyError, TypeError, ValueError) as exc:
        raise PlanError(f"malformed plan document: {exc}") from exc
    validate_plan(plan)
    return plan


def validate_plan(plan: EvaluationPlan) -> None:
    """Structural checks the kernels rely on (sizes, table ranges, group shapes)."""
    s = plan.s
    if len(plan.diag) != s or any(d <= 0 for d in plan.diag):
        raise PlanError("diag must have s positive entries")
    if not plan.shifts or any(len(sh) != s for sh in plan.shifts):
        raise PlanError("bad coset shifts")
    if plan.r < 1 or len(plan.sigma) != plan.r:
        raise PlanError("sigma table length must equal r")
    if any(v != SIGMA_SENTINEL and not 0 <= v < plan.N for v in plan.sigma):
        raise PlanError("sigma entry out of range")
    for n, _ in plan.planes:
        if len(n) != s:
            raise PlanError("plane normal length must equal s")
    for c in plan.classes:
        if not 0 <= c.kernel < plan.K:
            raise PlanError("class refers to a missing kernel")
        if len(c.T) != s or len(c.t) != s or len(c.pi_linear) != s or len(c.pi_offset) != s:
            raise PlanError("class transform has the wrong shape")
    for k in plan.kernels:
        for g in k.groups:
            if g.size not in (1, 2, 4, 8) or g.size != 1 << len(g.span_axes):
                raise PlanError("fetch group must have 2^len(span_axes) sites")
            if len(g.t_nums) != len(g.span_axes):
                raise PlanError("one t_num polynomial per span axis required")
            if any(len(site) != s for site in g.sites):
                raise PlanError("site length must equal s")


def canonical_body(doc: dict) -> str:
    return json.dumps(doc, sort_keys=True, separators=(",", ":"))


def serialize_plan(plan: EvaluationPlan) -> str:
    """plancompile.py:535-539 (same document, same checksum)."""
    doc = plan_to_dict(plan)
    checksum = hashlib.sha256(canonical_body(doc).encode()).hexdigest()
    return json.dumps({"checksum": checksum, "plan": doc}, sort_keys=True, indent=1)


def deserialize_plan(text: str) -> EvaluationPlan:
    """plancompile.py:542-557: checksum verified, format and version checked."""
    try:
        wrapper = json.loads(text)
    except json.JSONDecodeError as exc:
        raise PlanError(f"malformed plan document: {exc}") from exc
    if not isinstance(wrapper, dict) or "plan" not in wrapper or "checksum" not in wrapper:
        raise PlanError("plan document missing checksum or payload")
    doc = wrapper["plan"]
    digest = hashlib.sha256(canonical_body(doc).encode()).hexdigest()
    if digest != wrapper["checksum"]:
        raise PlanError("plan checksum mismatch")
    if doc.get("format") != _PLAN_FORMAT:
        raise PlanError("not an evaluation plan document")
    if doc.get("version") != _PLAN_VERSION:
        raise PlanError(f"unsupported plan version {doc.get('version')}")
    plan = plan_from_dict(doc)
    plan.checksum = digest
    return plan
