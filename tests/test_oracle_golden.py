"""CPU: the numpy oracle (oracle/plan_numpy.py) reproduces the REFERENCE's own outputs.

The golden fixtures were produced by running /root/reference (tests/golden/make_golden.py);
this pins the oracle before it is trusted as the checker for the GPU kernels.
"""
import numpy as np
import pytest

from conftest import golden_names, load_golden
from oracle.plan_numpy import NumpyGrid, PlanTables, classify_batch, eval_batch
from paper_2102_08514_b200.corpus import PLAN_DIR
from paper_2102_08514_b200.plan import deserialize_plan

NAMES = golden_names()


def _plan(name):
    return deserialize_plan((PLAN_DIR / f"{name}.plan.json").read_text())


def _grid(plan, g, boundary):
    arrays = [g[f"coset{k}"].astype(np.float64) for k in range(plan.M)]
    return NumpyGrid(plan.diag, plan.shifts, arrays, g["origins"], boundary)


@pytest.mark.parametrize("name", NAMES)
@pytest.mark.parametrize("boundary", ["zero", "clamp", "mirror"])
def test_oracle_matches_reference_batch(name, boundary):
    g = load_golden(name)
    plan = _plan(name)
    tabs = PlanTables(plan)
    got = eval_batch(plan, _grid(plan, g, boundary), g["pts"].astype(np.float64), tabs)
    ref = g[f"out_{boundary}"]
    # same float64 numpy operation sequence as runtime.py:363-408 -> bit-identical
    np.testing.assert_array_equal(got, ref)


@pytest.mark.parametrize("name", NAMES)
def test_oracle_classification_matches_reference(name):
    g = load_golden(name)
    plan = _plan(name)
    cls, cells = classify_batch(plan, g["pts"].astype(np.float64))
    np.testing.assert_array_equal(cls, g["classes"])
    np.testing.assert_array_equal(cells, g["cells"])
    assert (cls >= 0).all(), "no sigma sentinel is reachable from the fixtures"


@pytest.mark.parametrize("name", NAMES)
def test_reference_batch_agrees_with_bruteforce_and_scalar(name):
    """Pins the fixtures themselves: eval_batch vs eval_bruteforce (runtime.py:415-427)
    and vs the scalar program path (runtime.py:232-242), SPEC.md:476 (<= 1e-9)."""
    g = load_golden(name)
    sub = g["sub"]
    scale = max(1.0, float(np.max(np.abs(g["out_zero"]))))
    assert np.max(np.abs(g["scalar"] - g["out_zero"][sub])) <= 1e-9 * scale
    if np.isfinite(g["brute"]).all():
        assert np.max(np.abs(g["brute"] - g["out_zero"][sub])) <= 1e-9 * scale
    if np.isfinite(g["exact"]).all():
        # the exact rational convolution sum rounded once: the batch path is within ~1e-15
        assert np.max(np.abs(g["exact"] - g["out_zero"][sub])) <= 1e-14 * scale
