"""Plans compiled with non-default PlanOptions, derived natively from the catalog plan.

The reference compiles a plan per `PlanOptions(grouped, predicated, ordered,
texel_offset_half)` (plancompile.py:47-52, 339-380).  Only `grouped` and `ordered` change the
plan's content — the fetch groups of each kernel (`group_fetches` with grouped=False gives
singletons; `order_fetches` reorders) — `predicated` is recorded only and `texel_offset_half`
changes the lowered program's rounding (plancompile.py:696-697).  The classes, planes and sigma
are the same for every option set.  So the drop-in derives any option set from the default
catalog plan: each kernel's per-site weight polynomials are recovered exactly from its fetch
groups (corner weights of a rank-1 group: prod_j (t_num_j | g - t_num_j) / g^(k-1), an exact
polynomial division), then regrouped / reordered with the reference's rules (tpplan.py:
`group_fetches`, `order_fetches`, restatements of plancompile.py:150-325).  Checked against
plans the reference compiler produced with those options (tests/test_variants.py).
"""

from __future__ import annotations

from dataclasses import replace

from .exact import Poly
from .plan import EvaluationPlan, PlanKernel, PlanOptions

from .tpplan import group_fetches, order_fetches


def group_site_weights(group) -> list:
    """[(site, weight Poly)] of a fetch group (tensor-corner order over span_axes)."""
    k = len(group.span_axes)
    if k == 0:
        return [(tuple(group.sites[0]), group.g)]
    den = None
    for _ in range(k - 1):
        den = group.g if den is None else den * group.g
    out = []
    for idx, site in enumerate(group.sites):
        num = Poly.const(group.g.dim, 1)
        for j in range(k):
            num = num * (group.t_nums[j] if idx >> j & 1 else group.g - group.t_nums[j])
        out.append((tuple(site), num if den is None else num.divexact(den)))
    return out


def plan_variant(plan: EvaluationPlan, options: PlanOptions) -> EvaluationPlan:
    """The plan the reference compiler would emit for `options` (same analysis)."""
    grouped = options.grouped and plan.basis_nonnegative  # plancompile.py:350-351
    kernels = []
    for kern in plan.kernels:
        sw = sorted(sw for grp in kern.groups for sw in group_site_weights(grp))
        groups = group_fetches([s for s, _ in sw], [w for _, w in sw], plan.diag, grouped=grouped)
        if options.ordered:
            groups = order_fetches(groups, plan.diag)
        kernels.append(PlanKernel(kern.ref_class, tuple(groups)))
    return replace(plan, kernels=tuple(kernels), options=replace(options, grouped=grouped), checksum="")
