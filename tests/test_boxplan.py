"""Native box-spline plan producer (boxplan.py) against the reference compiler's output.

Anchors: the shipped catalog plans and PP documents (compiled by the reference, tools/
gen_plans.py / gen_pp.py) and tests/golden/boxplan/ (direction sets outside the catalog,
compiled by the reference end to end, tests/golden/make_boxplan_golden.py).  Equality is on
the full wire document (plan_to_dict), i.e. the same checksum.  The slow corpus members
(cc_tricubic 41 s, bcc_voronoi1 40 s, cc_zp3 36 s) run with SP_SLOW_TESTS=1; all of them
were checked equal.  bcc_quartic (DIAG + 2·E3): 720 pieces in 12 s here vs 252 s for the
reference's extraction, document byte-identical.
"""
import os

import pytest

from paper_2102_08514_b200 import boxplan, corpus, pp
from paper_2102_08514_b200.lattice import decompose_cartesian, named_lattice
from paper_2102_08514_b200.plan import PlanOptions, deserialize_plan, plan_to_dict

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = os.path.join(HERE, "golden", "boxplan")
SLOW = os.environ.get("SP_SLOW_TESTS") == "1"

E3 = [(1, 0, 0), (0, 1, 0), (0, 0, 1)]
GOLDEN_CASES = {
    "cc2_courant": ([(1, 0), (0, 1), (1, 1)], "CC2"),
    "cc2_biquadratic": ([(1, 0), (0, 1)] * 3, "CC2"),
    "qc_zp": ([(1, 0), (0, 1), (1, 1), (-1, 1)], "QC"),
    "cc2_hex3": ([(1, 0), (0, 1), (1, 1)] * 2, "CC2"),
    "cc3_e3_d1": (E3 + [(1, 1, 1)], "CC3"),
    "cc3_e3_d2": (E3 + [(1, 1, 1), (1, -1, 1)], "CC3"),
}

FAST = ["tp2", "zp", "qc_tensor", "cc_trilinear", "bcc_linear_rd", "bcc_quartic", "fcc_cubic", "bcc_quintic_rd"]
SLOW_NAMES = ["cc_tricubic"]


@pytest.mark.parametrize("name", FAST + [pytest.param(n, marks=pytest.mark.skipif(not SLOW, reason="SP_SLOW_TESTS"))
                                         for n in SLOW_NAMES])
def test_catalog_box_splines(name):
    cols, _ = corpus.direction_set(name)
    sp = boxplan.extract_pp_form(cols, name)
    assert pp.format_pp_spline(sp) == (corpus.PP_DIR / f"{name}.spp").read_text()
    lat, cos = corpus.lattice_of(name)
    plan = boxplan.compile_pp_plan(sp, lat, cos)
    assert plan_to_dict(plan) == plan_to_dict(corpus.build_plan(name))


@pytest.mark.parametrize("name", sorted(GOLDEN_CASES))
def test_golden_box_splines(name):
    cols, latname = GOLDEN_CASES[name]
    lat = named_lattice(latname)
    sp = boxplan.extract_pp_form(cols, name)
    with open(os.path.join(GOLD, f"{name}.spp")) as fh:
        assert pp.format_pp_spline(sp) == fh.read()
    plan = boxplan.compile_pp_plan(sp, lat, decompose_cartesian(lat))
    with open(os.path.join(GOLD, f"{name}.plan.json")) as fh:
        ref = deserialize_plan(fh.read())
    assert plan_to_dict(plan) == plan_to_dict(ref)


@pytest.mark.parametrize("name", ["fcc_voronoi1", pytest.param("bcc_voronoi1", marks=pytest.mark.skipif(
    not SLOW, reason="SP_SLOW_TESTS"))])
def test_voronoi_documents(name):
    """compile_pp_plan on an imported PP document (the Voronoi splines have no direction set)."""
    lat, cos = corpus.lattice_of(name)
    plan = boxplan.compile_pp_plan(corpus.build_spline(name, validate=False), lat, cos)
    assert plan_to_dict(plan) == plan_to_dict(corpus.build_plan(name))


@pytest.mark.skipif(not SLOW, reason="SP_SLOW_TESTS")
def test_zp3_ungrouped():
    cols, _ = corpus.direction_set("cc_zp3")
    lat, cos = corpus.lattice_of("cc_zp3")
    opts = PlanOptions(grouped=False)
    plan = boxplan.box_spline_plan(cols, lat, cos, "cc_zp3", opts)
    assert plan_to_dict(plan) == plan_to_dict(corpus.build_plan("cc_zp3", opts))


def test_options_variants_match_regrouping():
    """Other PlanOptions compiled natively equal the catalog-derived variants (variants.py)."""
    cols, _ = corpus.direction_set("bcc_linear_rd")
    lat, cos = corpus.lattice_of("bcc_linear_rd")
    for opts in (PlanOptions(grouped=False), PlanOptions(ordered=False)):
        plan = boxplan.box_spline_plan(cols, lat, cos, "bcc_linear_rd", opts)
        assert plan_to_dict(plan) == plan_to_dict(corpus.build_plan("bcc_linear_rd", opts))


def test_not_a_partition_of_unity_is_refused():
    """E3 x 2 on FCC: the reference raises in enumerate_subregions (analysis.py:124)."""
    lat = named_lattice("FCC")
    with pytest.raises(pp.SplineError):
        boxplan.box_spline_plan(E3 * 2, lat, decompose_cartesian(lat), "fcc_trilinear")


def test_pp_form_values_match_recurrence():
    """Piece polynomials equal the box-spline recurrence at points off the knot planes."""
    from fractions import Fraction

    cols = [(1, 0), (0, 1), (1, 1), (-1, 1)]
    sp = boxplan.extract_pp_form(cols, "zp")
    rec = boxplan._BoxRecurrence([tuple(Fraction(v) for v in c) for c in cols])
    for x in [(Fraction(1, 3), Fraction(5, 7)), (Fraction(-2, 5), Fraction(3, 2)), (Fraction(1, 11), Fraction(1, 13))]:
        assert sp.eval_exact(x) == rec.piece(x).eval(list(x))
