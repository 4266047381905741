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
