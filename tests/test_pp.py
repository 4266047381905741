"""CPU: the spline-selection API (corpus.build_spline / build_pair, pp.py) against the
REFERENCE: shipped PP documents round-trip byte for byte through our parser / formatter, and
exact point values and contributing sites equal the reference's own (frozen by
tests/golden/make_pp_golden.py)."""
import json
import os
from fractions import Fraction

import pytest

from paper_2102_08514_b200 import corpus, pp

HERE = os.path.dirname(os.path.abspath(__file__))
REF = json.load(open(os.path.join(HERE, "golden", "pp_values.json")))


@pytest.mark.parametrize("name", sorted(REF))
def test_document_round_trip(name):
    text = (corpus.PP_DIR / f"{name}.spp").read_text()
    sp = pp.import_pp_spline(text, validate=False)
    assert len(sp.pieces) == REF[name]["pieces"]
    assert pp.format_pp_spline(sp) == text


@pytest.mark.parametrize("name", [n for n in sorted(REF) if REF[n]["pieces"] <= 400])
def test_exact_values_and_sites_match_reference(name):
    sp = pp.import_pp_spline((corpus.PP_DIR / f"{name}.spp").read_text(), validate=False)
    r = REF[name]
    for p, v in zip(r["points"], r["values"]):
        assert sp.eval_exact([Fraction(c) for c in p]) == Fraction(v), (name, p)
    if name in corpus.DIRECTION_SETS or name in corpus.VORONOI_SPLINES:
        lat, cos = corpus.lattice_of(name)
        sol = pp.SplineOnLattice(sp, lat, cos)
        for p, sites in zip(r["points"][-4:], r["sites"]):
            assert sol.contributing_sites([Fraction(c) for c in p]) == [tuple(s) for s in sites]


@pytest.mark.parametrize("name", ["bcc_linear_rd", "fcc_cubic", "fcc_voronoi1", "cc_trilinear"])
def test_build_pair_partition_of_unity(name):
    sol = corpus.build_pair(name)  # validate=True: degree bound, bounded pieces, PoU, sign
    pts = [(Fraction(3, 7), Fraction(-5, 11), Fraction(9, 13)), (Fraction(1, 2), Fraction(1, 2), Fraction(0))]
    for x in pts:
        assert sol.partition_of_unity_at(x) == 1


def test_build_spline_errors(tmp_path):
    with pytest.raises(KeyError):
        corpus.build_spline("no_such_spline")
    with pytest.raises(pp.SplineError):
        pp.import_pp_spline("not a document")
    bad = (corpus.PP_DIR / "cc_trilinear.spp").read_text().replace("degree 3", "degree 1")
    with pytest.raises(pp.SplineError):
        pp.import_pp_spline(bad, validate=False)
