"""Approximation-order harness: the GPU
reconstruction must reach each spline's published order (paper Table 1,
corpus.REFERENCE_ORDERS) on a smooth target, reproduce constants (partition of unity,
SPEC.md:516), and the BCC quintic spline reaches order 4 only WITH its quasi-interpolation
prefilter (corpus.py:71-82) — an end-to-end check of plan kernels + prefilter at scale."""
import numpy as np
import pytest
import torch

from paper_2102_08514_b200 import corpus
from paper_2102_08514_b200.convergence import _fit_order, constant, gaussian, run_convergence, spline_center


def test_fit_order_and_centres():
    hs = [0.25, 0.125, 0.0625]
    assert abs(_fit_order(hs, [h ** 3 * 7 for h in hs]) - 3.0) < 1e-9
    assert spline_center(corpus.build_plan("cc_trilinear")) == (1.0, 1.0, 1.0)
    assert spline_center(corpus.build_plan("bcc_quintic_rd")) == (2.0, 2.0, 2.0)
    assert spline_center(corpus.load_plan(corpus.PLAN_DIR / "cc_zp3_ungrouped.plan.json")) == (1.5, 1.5, 1.5)


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["cc_trilinear", "cc_tricubic", "bcc_linear_rd", "fcc_cubic"])
def test_constant_is_reproduced(name, cuda):
    plan = corpus.build_plan(name) if name in corpus.DIRECTION_SETS and name != "cc_tricubic" else \
        corpus.load_plan(corpus.PLAN_DIR / f"{name}.plan.json")
    rep = run_convergence(plan, constant(0.7), halvings=2, samples=200_000, device=cuda)
    assert max(rep.max_errors) < 1e-12


def cubic_bspline_quasi_interpolant():
    """Tensor-product cubic B-spline quasi-interpolation taps (1-D [-1/6, 4/3, -1/6]):
    1/B-hat(w) = 1 + w^2/6 + O(w^4) matched by a 3-tap stencil per axis (27 taps)."""
    one = {-1: -1.0 / 6.0, 0: 4.0 / 3.0, 1: -1.0 / 6.0}
    return {(a, b, c): one[a] * one[b] * one[c] for a in one for b in one for c in one}


# Sampling without a prefilter reproduces only the second-order terms of a symmetric
# spline: every spline converges at order 2 (min(order, 2)); with the quasi-interpolation
# prefilter it reaches its Table-1 order (bcc_quintic_rd: the reference's taps; tricubic:
# the classical cubic B-spline taps, also exercising the 27-tap stencil).
@pytest.mark.gpu
@pytest.mark.parametrize("name,order,taps", [
    ("cc_trilinear", 2, None), ("bcc_linear_rd", 2, None), ("fcc_cubic", 2, None), ("cc_tricubic", 2, None),
    ("bcc_quintic_rd", 2, None), ("bcc_quintic_rd", 4, "reference"), ("cc_tricubic", 4, "cubic")])
def test_approximation_order(name, order, taps, cuda):
    plan = corpus.load_plan(corpus.PLAN_DIR / f"{name}.plan.json")
    pre = {None: None, "reference": corpus.prefilter_taps(name) if taps == "reference" else None,
           "cubic": cubic_bspline_quasi_interpolant()}[taps]
    rep = run_convergence(plan, gaussian(), prefilter=pre, h0=0.125, halvings=4, samples=400_000, device=cuda)
    assert np.all(np.diff(rep.errors) < 0), rep.errors
    assert abs(rep.fitted_order - order) < 0.35, (rep.fitted_order, rep.errors)
    if order == 4:
        assert corpus.REFERENCE_ORDERS.get(name, 4) == 4


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["tp2", "zp", "qc_tensor"])
def test_two_dimensional_corpus_splines(name, cuda):
    """SPEC.md convergence examples in 2-D: TP2 on CC with a Gaussian target converges at
    order 2; constants are reproduced (the 2-D plans run through their 3-D lift)."""
    plan = corpus.build_plan(name)
    rep = run_convergence(plan, constant(0.3), halvings=2, samples=100_000, device=cuda)
    assert max(rep.max_errors) < 1e-12
    rep = run_convergence(plan, gaussian(sigma=0.125), h0=0.0625, halvings=4, samples=200_000, device=cuda)
    assert np.all(np.diff(rep.errors) < 0), rep.errors
    assert abs(rep.fitted_order - corpus.REFERENCE_ORDERS.get(name, 2)) < 0.35, (rep.fitted_order, rep.errors)
