"""CPU: plans for non-default PlanOptions derived natively from the catalog plan
(variants.plan_variant, corpus.build_plan(name, options)) equal the plans the REFERENCE
compiler emits for those options (checksums frozen by tests/golden/make_variant_golden.py)."""
import json
import os

import pytest

from paper_2102_08514_b200 import corpus
from paper_2102_08514_b200.plan import PlanOptions, serialize_plan

HERE = os.path.dirname(os.path.abspath(__file__))
REF = json.load(open(os.path.join(HERE, "golden", "variants.json")))


def _opts(key):
    kw = {}
    for item in key.split(":")[1].split(","):
        k, v = item.split("=")
        kw[k] = v == "True"
    return PlanOptions(**kw)


@pytest.mark.parametrize("key", sorted(REF))
def test_variant_matches_reference_compile(key):
    name = key.split(":")[0]
    plan = corpus.build_plan(name, _opts(key))
    assert json.loads(serialize_plan(plan))["checksum"] == REF[key], key
