"""CPU: the IR seam (PlanInterpreter.program / emit_kernel / parse_kernel / execute) against
the REFERENCE: rendered programs identical to the reference's emit_kernel (digests made by
tests/golden/make_program_golden.py), and execute() on the golden grids bit-identical to the
reference's scalar PlanInterpreter.eval outputs (runtime.py:232-242) frozen in the goldens."""
import hashlib
import json
import os

import numpy as np
import pytest

from conftest import load_golden
from paper_2102_08514_b200 import corpus
from paper_2102_08514_b200.minilang import build_program, emit_kernel, execute, parse_kernel
from paper_2102_08514_b200.runtime import PlanInterpreter

HERE = os.path.dirname(os.path.abspath(__file__))
DIGESTS = json.load(open(os.path.join(HERE, "golden", "programs.json")))


@pytest.mark.parametrize("name", sorted(DIGESTS))
def test_program_text_is_the_references(name):
    plan = corpus.load_plan(corpus.PLAN_DIR / f"{name}.plan.json")
    text = emit_kernel(plan)
    want = DIGESTS[name]
    assert len(build_program(plan).ops) == want["ops"]
    assert hashlib.sha256(text.encode()).hexdigest() == want["sha256"]
    # parse(render(p)) renders to the same document
    assert parse_kernel(text).render() == text


def _host_grid(plan, g, boundary):
    """The golden grid as a host CoefficientGrid: its fetch_nearest / fetch_linear are the
    reference's scalar accessors (runtime.py:125-147)."""
    from paper_2102_08514_b200.lattice import decompose_cartesian, named_lattice
    from paper_2102_08514_b200.runtime import CoefficientGrid

    cos = decompose_cartesian(named_lattice(plan.lattice_name))
    arrays = [g[f"coset{k}"].astype(np.float64) for k in range(plan.M)]
    return CoefficientGrid(cos, arrays, [tuple(o) for o in g["origins"]], boundary, device="cpu")


@pytest.mark.parametrize("name", ["cc_trilinear", "bcc_linear_rd", "fcc_cubic", "bcc_quintic_rd", "fcc_voronoi1",
                                  "cc_tricubic"])
def test_execute_matches_reference_scalar_eval(name):
    g = load_golden(name)
    plan = corpus.load_plan(corpus.PLAN_DIR / f"{name}.plan.json")
    prog = PlanInterpreter(plan).program()
    grid = _host_grid(plan, g, "zero")
    half = plan.options.texel_offset_half
    got = np.array([execute(prog, [float(v) for v in g["pts"][i].astype(np.float64)], grid.fetch_nearest,
                            lambda k, u: grid.fetch_linear(k, u, offset_half=half))
                    for i in g["sub"]])
    np.testing.assert_array_equal(got, g["scalar"])
