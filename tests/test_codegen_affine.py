"""Affine plans (codegen.affine_tables): the per-plane-code coefficient table must equal the
plan's weight polynomials composed with the class transform y = T xp - t (runtime.py:385),
exactly, for every code q — including the sigma sentinel, evaluated as class 0 and flagged."""
from fractions import Fraction

import numpy as np

from paper_2102_08514_b200 import codegen, corpus


def test_affine_table_is_the_composed_polynomials():
    plan = corpus.build_plan("bcc_linear_rd")
    rows, mask = codegen.affine_tables(plan)
    polys = []
    for g in plan.kernels[0].groups:
        polys.append(g.g)
        polys.extend(g.t_nums)
    rng = np.random.default_rng(0)
    assert len(rows) == plan.r
    for q, row in enumerate(rows):
        c = plan.sigma[q]
        assert bool(mask >> q & 1) == (c < 0)
        ct = plan.classes[max(c, 0)]
        for _ in range(3):
            xp = [Fraction(int(v), 64) for v in rng.integers(0, 128, 3)]
            y = [sum(Fraction(ct.T[i][j]) * xp[j] for j in range(3)) - Fraction(ct.t[i]) for i in range(3)]
            for poly, (a0, a1, a2, cc) in zip(polys, row):
                want = sum(Fraction(coef) * (y[e.index(1)] if sum(e) else 1) for e, coef in poly.terms.items())
                assert a0 * xp[0] + a1 * xp[1] + a2 * xp[2] + cc == want


def test_affine_only_for_degree_one_single_kernel_plans():
    assert codegen.affine_tables(corpus.build_plan("bcc_quintic_rd")) is None
    assert codegen.affine_tables(corpus.build_plan("fcc_cubic")) is None
    src, stats = codegen.generate_plan_source(corpus.build_plan("bcc_linear_rd"), "bcc_linear_rd")
    assert stats["affine"] and "kernel_aff" in src and "kAff" in src
