"""Native tensor-product plan producer (tpplan.py) vs the reference
compiler: the produced plan document must be byte-identical — same canonical JSON, same
sha256 checksum — to plans the reference compiled (plancompile.py:328-380 + serialize_plan):
cc_trilinear / cc_tricubic from the catalog, cc_tp2 (and cc_tp4 when frozen) from
tests/golden/tp_plans/ (tests/golden/make_tp_plans.py).  GPU: the plans evaluate like the
oracle."""
import json
import pathlib

import numpy as np
import pytest
import torch

from paper_2102_08514_b200 import corpus
from paper_2102_08514_b200.exact import tensor_site_weight
from paper_2102_08514_b200.plan import PlanOptions, serialize_plan
from paper_2102_08514_b200.tpplan import group_fetches, tensor_product_plan

GOLD = pathlib.Path(__file__).parent / "golden" / "tp_plans"

CASES = [(1, corpus.PLAN_DIR / "cc_trilinear.plan.json", "cc_trilinear"),
         (3, corpus.PLAN_DIR / "cc_tricubic.plan.json", "cc_tricubic")]
CASES += [(int(p.stem.split(".")[0][5:]), p, p.stem.split(".")[0]) for p in sorted(GOLD.glob("cc_tp*.plan.json"))]


@pytest.mark.parametrize("degree,path,name", CASES, ids=[c[2] for c in CASES])
def test_plan_document_identical_to_reference(degree, path, name):
    mine = serialize_plan(tensor_product_plan(degree, name))
    ref = path.read_text()
    assert json.loads(mine)["checksum"] == json.loads(ref)["checksum"]
    assert mine == ref


def test_build_plan_family_and_degree_proof():
    p = corpus.build_plan("cc_tp2")
    assert p.name == "cc_tp2" and p.tensor_bspline_degree() == 2
    assert p.kernels[0].nearest_count == 27 and len(p.kernels[0].groups) == 8
    assert corpus.lattice_of("cc_tp5")[1].M == 1
    ung = tensor_product_plan(2, options=PlanOptions(grouped=False))
    assert all(g.size == 1 for g in ung.kernels[0].groups) and ung.kernels[0].nearest_count == 27
    assert ung.tensor_bspline_degree() == 2


def test_general_grouping_matches_tensor_fast_path():
    """group_fetches (rank-1 identities checked on the polynomials) == the closed form."""
    from itertools import product

    sites = sorted(product(range(-2, 1), repeat=3))
    gen = group_fetches(sites, [tensor_site_weight(2, 3, s) for s in sites], (1, 1, 1))
    assert gen == tuple(sorted(tensor_product_plan(2, options=PlanOptions(ordered=False)).kernels[0].groups,
                               key=lambda g: (-g.size, g.sites)))


@pytest.mark.gpu
@pytest.mark.parametrize("degree", [0, 2, 4])
def test_tensor_plans_evaluate_like_the_oracle(degree, cuda):
    from oracle.plan_numpy import NumpyGrid, PlanTables, eval_batch as oracle_eval
    from paper_2102_08514_b200.runtime import CoefficientGrid, PlanInterpreter

    plan = tensor_product_plan(degree)
    _, cos = corpus.lattice_of(plan.name)
    rng = np.random.default_rng(degree)
    arr = rng.random((20, 20, 20))
    grid = CoefficientGrid(cos, [torch.from_numpy(arr)], [(0, 0, 0)], "mirror", device=cuda, dtype=torch.float64)
    pts = rng.uniform(-2, 22, size=(3000, 3))
    interp = PlanInterpreter(plan)
    got = interp.eval_batch(grid, torch.from_numpy(pts).to(cuda)).cpu().numpy()
    ref = oracle_eval(plan, NumpyGrid(plan.diag, plan.shifts, [arr], [(0, 0, 0)], "mirror"), pts, PlanTables(plan))
    assert np.abs(got - ref).max() <= 1e-12 * np.abs(ref).max()
    ones = CoefficientGrid(cos, [torch.ones(20, 20, 20, dtype=torch.float64)], [(0, 0, 0)], "clamp", device=cuda)
    pou = interp.eval_batch(ones, torch.from_numpy(pts).to(cuda))
    assert float((pou - 1).abs().max()) < 1e-12


def _exhaustive_cover(n, rows):
    """The reference's search (plancompile.py:233-268) restated as the checker: every exact
    cover, smallest cardinality, then least sorted tuple of sorted rows."""
    best = None
    by_elem = {e: [i for i, r in enumerate(rows) if e in r] for e in range(n)}

    def dfs(left, chosen):
        nonlocal best
        if not left:
            key = (len(chosen), tuple(sorted(tuple(sorted(rows[i])) for i in chosen)))
            if best is None or key < best[0]:
                best = (key, list(chosen))
            return
        e = min(left, key=lambda e: (sum(1 for i in by_elem[e] if rows[i] <= left), e))
        for i in by_elem[e]:
            if rows[i] <= left:
                chosen.append(i)
                dfs(left - rows[i], chosen)
                chosen.pop()

    dfs(frozenset(range(n)), [])
    return best[1]


def test_min_exact_cover_matches_exhaustive_search():
    """The fast cover (fractional bound + greedy least key) returns the reference's cover on
    random instances with many tied minimum covers."""
    import random

    from paper_2102_08514_b200.tpplan import _min_exact_cover

    rng = random.Random(5)
    for _ in range(300):
        n = rng.randint(1, 12)
        rows = {frozenset([e]) for e in range(n)}
        for _ in range(rng.randint(0, 3 * n)):
            k = rng.choice([2, 2, 4, 4, 8])
            if k <= n:
                rows.add(frozenset(rng.sample(range(n), k)))
        rows = sorted(rows, key=lambda r: (len(r), sorted(r)))
        rng.shuffle(rows)
        got = _min_exact_cover(n, rows)
        want = _exhaustive_cover(n, rows)
        key = lambda c: tuple(sorted(tuple(sorted(rows[i])) for i in c))  # noqa: E731
        assert len(got) == len(want) and key(got) == key(want)


def test_grouped_zp3_resolves():
    """build_plan('cc_zp3') with default options: 53 sites per kernel grouped exactly."""
    plan = corpus.build_plan("cc_zp3")
    assert plan.options.grouped
    for k in plan.kernels:
        sites = sorted(s for g in k.groups for s in g.sites)
        assert len(sites) == len(set(sites)) == 53
    assert plan.grouped_fetch_counts()[0] < plan.nearest_fetch_counts()[0]
