"""CPU: plan loading, wire format, specialisation analysis, lattice KATs, codegen."""
import json
from fractions import Fraction

import numpy as np
import pytest

from paper_2102_08514_b200 import corpus
from paper_2102_08514_b200.codegen import codegen_supported, generate_plan_source
from paper_2102_08514_b200.exact import Poly, bspline_piece_polys, horner_tree, tensor_site_weight
from paper_2102_08514_b200.lattice import decompose_cartesian, named_lattice, parse_lattice_file, rho
from paper_2102_08514_b200.packing import canonical_words, pack_plan
from paper_2102_08514_b200.plan import PlanError, deserialize_plan, serialize_plan

CATALOG = corpus.available_plans()


@pytest.mark.parametrize("name", CATALOG)
def test_plan_roundtrip_and_checksum(name):
    text = (corpus.PLAN_DIR / f"{name}.plan.json").read_text()
    plan = deserialize_plan(text)
    again = deserialize_plan(serialize_plan(plan))
    assert again == plan
    # the reference's checksum (plancompile.py:535-539) is reproduced exactly
    assert json.loads(serialize_plan(plan))["checksum"] == json.loads(text)["checksum"]


def test_checksum_mismatch_rejected():
    text = (corpus.PLAN_DIR / "bcc_linear_rd.plan.json").read_text()
    doc = json.loads(text)
    doc["plan"]["sigma"][0] = 3
    with pytest.raises(PlanError):
        deserialize_plan(json.dumps(doc))
    with pytest.raises(PlanError):
        deserialize_plan("{not json")


def test_table1_lookup_counts():
    """Table 1 / corpus.py:52-57: nearest lookups per reconstruction."""
    for name, want in corpus.REFERENCE_LOOKUPS.items():
        if name not in CATALOG:
            name_u = f"{name}_ungrouped"
            if name_u not in CATALOG:
                continue
            name = name_u
        plan = corpus.load_plan(corpus.PLAN_DIR / f"{name}.plan.json")
        assert set(plan.nearest_fetch_counts()) == {want}, name


def test_known_plan_shapes():
    """SPEC.md:302-304, SURVEY.md §9 plan statistics."""
    p = corpus.build_plan("zp")
    assert (p.N, p.Q, p.r, p.K) == (4, 2, 4, 1)
    p = corpus.build_plan("bcc_quartic")
    assert p.Q == 9
    p = corpus.build_plan("fcc_cubic")
    assert (p.M, p.N, p.Q, p.r, p.K) == (4, 40, 11, 180, 3)
    p = corpus.build_plan("bcc_quintic_rd")
    assert (p.M, p.N, p.Q, p.r, p.K) == (2, 24, 6, 64, 1)


def test_tensor_bspline_detection():
    assert corpus.build_plan("cc_trilinear").tensor_bspline_degree() == 1
    assert corpus.build_plan("cc_tricubic").tensor_bspline_degree() == 3
    for name in ("bcc_linear_rd", "fcc_cubic", "zp"):
        assert corpus.build_plan(name).tensor_bspline_degree() is None


def test_bspline_pieces_partition_of_unity():
    for deg in (1, 2, 3):
        pieces = bspline_piece_polys(deg)
        total = [Fraction(0)] * (deg + 1)
        for p in pieces:
            for k, c in enumerate(p):
                total[k] += c
        assert total == [Fraction(1)] + [Fraction(0)] * deg
    # cubic B-spline at t = 1/2 on its four pieces: 1/48, 23/48, 23/48, 1/48
    half = [Fraction(1, 2)] * 3
    assert tensor_site_weight(3, 3, (0, 0, 0)).eval(half) == Fraction(1, 48) ** 3
    assert tensor_site_weight(3, 3, (-1, -2, -3)).eval(half) == Fraction(23, 48) ** 2 * Fraction(1, 48)
    assert tensor_site_weight(3, 3, (1, 0, 0)).eval(half) == 0


def test_horner_tree_exact():
    rng = np.random.default_rng(5)
    for _ in range(20):
        terms = {}
        for _ in range(8):
            e = tuple(int(v) for v in rng.integers(0, 4, size=3))
            terms[e] = Fraction(int(rng.integers(-9, 10)), int(rng.integers(1, 7)))
        p = Poly(3, terms)
        tree = horner_tree(p)
        pt = [Fraction(int(rng.integers(-5, 6)), 3) for _ in range(3)]

        def ev(n):
            if n.kind == "const":
                return n.args[0]
            if n.kind == "var":
                return pt[n.args[0]]
            a = [ev(x) for x in n.args]
            return a[0] + a[1] if n.kind == "add" else (a[0] * a[1] if n.kind == "mul" else a[0] * a[1] + a[2])

        assert ev(tree) == p.eval(pt)


@pytest.mark.parametrize("name", CATALOG)
def test_signed_permutation_classes_and_reach(name):
    plan = corpus.load_plan(corpus.PLAN_DIR / f"{name}.plan.json")
    recs = plan.signed_permutation_classes()
    assert recs is not None  # probe12: every corpus T/piA is a signed permutation
    for r, c in zip(recs, plan.classes):
        # piA == T^-1 (analysis.py:366 first candidate)
        T = np.array([[float(v) for v in row] for row in c.T])
        A = np.array(c.pi_linear, dtype=float)
        assert np.allclose(A @ T, np.eye(plan.s))
    lo, hi = plan.site_reach()
    assert all(a <= b for a, b in zip(lo, hi))


def test_codegen_sources():
    for name in CATALOG:
        plan = corpus.load_plan(corpus.PLAN_DIR / f"{name}.plan.json")
        if codegen_supported(plan):
            src, stats = generate_plan_source(plan, name)
            assert f"kGen_{stats['ident']}" in src
            assert stats["words"] == len(canonical_words(pack_plan(plan)))


def test_lattice_kats():
    """SPEC.md:102-113."""
    c = decompose_cartesian(named_lattice("BCC"))
    assert c.diag == (2, 2, 2) and c.shifts == ((0, 0, 0), (1, 1, 1))
    c = decompose_cartesian(named_lattice("FCC"))
    assert c.diag == (2, 2, 2) and c.shifts == ((0, 0, 0), (0, 1, 1), (1, 0, 1), (1, 1, 0))
    c = decompose_cartesian(named_lattice("QC"))
    assert c.diag == (2, 2) and c.shifts == ((0, 0), (1, 1))
    assert rho((2.5, 3.5), (2, 2)) == (2, 2)
    assert rho((-0.25, -0.25), (2, 2)) == (-2, -2)
    assert rho((Fraction(5, 2), Fraction(7, 2)), (2, 2)) == (2, 2)
    lat = parse_lattice_file("3\n-1 1 1\n1 -1 1\n1 1 -1\n", "bcc")
    assert lat.det() == 4
    c = decompose_cartesian(lat)
    assert c.index_of((3, 1, 1)).coset == 1 and c.site_of(c.index_of((3, 1, 1))) == (3, 1, 1)


def test_grid_extents_match_reference_rule():
    from paper_2102_08514_b200.runtime import grid_extents

    c = decompose_cartesian(named_lattice("BCC"))
    origins, shapes = grid_extents(c, [0, 0, 0], [405, 405, 405])
    assert shapes == [(203, 203, 203), (203, 203, 203)]
    assert sum(int(np.prod(s)) for s in shapes) == 16_730_854
    c = decompose_cartesian(named_lattice("FCC"))
    origins, shapes = grid_extents(c, [0, 0, 0], [321, 321, 321])
    assert sum(int(np.prod(s)) for s in shapes) == 16_693_124


@pytest.mark.parametrize("boundary", ["zero", "clamp", "mirror"])
def test_scalar_fetches_match_oracle(boundary):
    """CoefficientGrid.fetch_nearest / fetch_linear (runtime.py:125-147) against the oracle's
    batch fetches (runtime.py:170-188) on a BCC grid, in and outside storage."""
    import numpy as np
    import torch

    from oracle.plan_numpy import NumpyGrid
    from paper_2102_08514_b200.lattice import decompose_cartesian, named_lattice
    from paper_2102_08514_b200.runtime import CoefficientGrid

    cos = decompose_cartesian(named_lattice("BCC"))
    grid = CoefficientGrid.zeros(cos, [-3, -2, -1], [6, 5, 7], boundary=boundary, device="cpu",
                                 dtype=torch.float64)
    rng = np.random.default_rng(4)
    for a in grid.arrays:
        a.copy_(torch.from_numpy(rng.random(tuple(a.shape))))
    ng = NumpyGrid(cos.diag, cos.shifts, [a.numpy() for a in grid.arrays], grid.origins, boundary)
    z = rng.uniform(-6, 9, size=(200, 3))
    z[:20] = np.round(z[:20]) + 0.5  # half-way ties: round half to even
    for k in range(cos.M):
        want_n = ng.fetch_nearest_batch(k, z)
        want_l = ng.fetch_linear_batch(k, z)
        got_n = [grid.fetch_nearest(k, tuple(p)) for p in z]
        got_l = [grid.fetch_linear(k, tuple(p)) for p in z]
        np.testing.assert_array_equal(got_n, want_n)
        np.testing.assert_allclose(got_l, want_l, rtol=1e-14, atol=1e-15)
        half = [grid.fetch_linear(k, tuple(p + 0.5), offset_half=True) for p in z]
        np.testing.assert_allclose(half, want_l, rtol=1e-13, atol=1e-14)


def test_choose_order_heuristic():
    """eval_batch(order="auto") routing: iid points -> sort (protocol B), Morton-sorted ->
    morton (protocol A), raster scans / ray slabs (coherent) -> given (chunk staging)."""
    import torch

    from paper_2102_08514_b200.runtime import _morton64, choose_order

    rng = np.random.default_rng(0)
    iid = torch.from_numpy(rng.uniform(0, 200, (300_000, 3)))
    assert choose_order(iid) == "sort"
    keys = _morton64(np.floor(iid.numpy()).astype(np.int64))
    assert choose_order(iid[torch.from_numpy(np.argsort(keys, kind="stable"))]) == "morton"
    g = torch.arange(64, dtype=torch.float64)
    raster = torch.stack(torch.meshgrid(g, g, g, indexing="ij"), -1).reshape(-1, 3) + 0.5
    assert choose_order(raster) in ("given", "morton")
    rays = (torch.arange(1000, dtype=torch.float64)[:, None, None] * torch.tensor([0.0, 0.0, 0.0])
            + torch.from_numpy(rng.uniform(0, 100, (1000, 1, 3)))
            + torch.linspace(0, 50, 300, dtype=torch.float64)[None, :, None] * torch.tensor([0.3, 0.5, 0.8]))
    assert choose_order(rays.reshape(-1, 3)) == "given"
    assert choose_order(iid[:1]) == "given"


def test_choose_order_sample_indices_stay_in_range():
    """Sampling indices are exact integers for any batch size (a float32 linspace rounded
    n - 2 up to n for n = 1e8): a large strided view keeps the memory small."""
    import torch

    from paper_2102_08514_b200.runtime import choose_order

    big = (torch.rand(1, 3, dtype=torch.float64) * 50).expand(100_000_000, 3)  # 1e8 rows, stride-0 view
    assert choose_order(big) == "morton"  # identical points: every pair is non-decreasing


def test_eval_batch_unordered_rejects_host_inputs():
    """eval_batch_unordered (protocol B, values in brick order + permutation) has no CPU
    host fallback: non-tensor and wrongly shaped points are refused loudly."""
    import torch

    from paper_2102_08514_b200 import corpus
    from paper_2102_08514_b200.runtime import CoefficientGrid, PlanInterpreter, RuntimeError_

    plan = corpus.build_plan("cc_trilinear")
    _, cos = corpus.lattice_of("cc_trilinear")
    grid = CoefficientGrid.zeros(cos, [0, 0, 0], [7, 7, 7], device="cpu", dtype=torch.float32)
    interp = PlanInterpreter(plan)
    with pytest.raises(RuntimeError_):
        interp.eval_batch_unordered(grid, torch.zeros(4, 2))
    with pytest.raises(RuntimeError_):
        interp.eval_batch_unordered(grid, np.zeros((4, 3)))
