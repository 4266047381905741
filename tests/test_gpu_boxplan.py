"""Plans produced natively (boxplan.py) for direction sets outside the catalog, evaluated on the
GPU: the whole drop-in pipeline — direction matrix -> PP form -> plan -> sp_eval — against the
numpy oracle (oracle/plan_numpy.py, runtime.py:363-408 restated) on the same plan.  The plans
themselves equal the reference compiler's (tests/test_boxplan.py, tests/golden/boxplan/)."""
import numpy as np
import pytest
import torch

from oracle.plan_numpy import NumpyGrid, PlanTables, eval_batch as oracle_eval
from paper_2102_08514_b200 import boxplan
from paper_2102_08514_b200.lattice import decompose_cartesian, named_lattice
from paper_2102_08514_b200.runtime import CoefficientGrid, PlanInterpreter

pytestmark = pytest.mark.gpu

E3 = [(1, 0, 0), (0, 1, 0), (0, 0, 1)]
CASES = {
    "cc2_courant": ([(1, 0), (0, 1), (1, 1)], "CC2"),
    "qc_zp": ([(1, 0), (0, 1), (1, 1), (-1, 1)], "QC"),
    "cc2_hex3": ([(1, 0), (0, 1), (1, 1)] * 2, "CC2"),
    "cc3_e3_d1": (E3 + [(1, 1, 1)], "CC3"),
    "cc3_e3_d2": (E3 + [(1, 1, 1), (1, -1, 1)], "CC3"),
}


@pytest.mark.parametrize("name", sorted(CASES))
@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_native_plan_on_gpu_matches_oracle(name, dtype, cuda):
    cols, latname = CASES[name]
    lat = named_lattice(latname)
    cos = decompose_cartesian(lat)
    plan = boxplan.box_spline_plan(cols, lat, cos, name)
    s = plan.s
    lo, hi = [0] * s, [12] * s
    grid = CoefficientGrid.zeros(cos, lo, hi, boundary="clamp", device=cuda, dtype=dtype)
    gen = torch.Generator(device=cuda).manual_seed(11)
    for a in grid.arrays:
        a.copy_(torch.rand(a.shape, generator=gen, device=cuda, dtype=torch.float64).to(dtype))
    rng = np.random.default_rng(5)
    pts = rng.uniform(-2, 14, size=(20_000, s))
    interp = PlanInterpreter(plan)
    got = interp.eval_batch(grid, torch.from_numpy(pts).to(cuda, dtype)).double().cpu().numpy()
    ngrid = NumpyGrid(plan.diag, plan.shifts, [a.double().cpu().numpy() for a in grid.arrays], grid.origins, "clamp")
    ptsd = torch.from_numpy(pts).to(dtype).double().numpy()  # the points the kernel saw
    ref = oracle_eval(plan, ngrid, ptsd, PlanTables(plan))
    tol = 1e-12 if dtype == torch.float64 else 1e-5
    assert np.abs(got - ref).max() <= tol * max(1.0, np.abs(ref).max()), interp.kernel_name()
