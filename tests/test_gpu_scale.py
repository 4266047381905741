"""GPU, BASELINE sizes: size-independent properties + oracle spot checks on subsamples."""
import numpy as np
import pytest
import torch

from oracle.plan_numpy import NumpyGrid, PlanTables, eval_batch as oracle_eval
from paper_2102_08514_b200 import corpus
from paper_2102_08514_b200.runtime import CoefficientGrid, PlanInterpreter, morton_order

pytestmark = pytest.mark.gpu

CONFIGS = {  # C1, C2, C3, C4 (ZP3, FCC-6), C5 (Voronoi at 512^3-equivalent samples)
    "cc_trilinear": 63,
    "cc_tricubic": 255,
    "bcc_linear_rd": 405,
    "bcc_quintic_rd": 405,
    "fcc_cubic": 321,
    "cc_zp3": 255,
    "fcc_voronoi1": 643,
    "bcc_voronoi1": 811,
}


def _load_plan(name):
    """The catalog plan of a BASELINE spline (cc_zp3 ships as its PlanOptions(grouped=False)
    compilation when the grouped one is not in the catalog)."""
    names = corpus.available_plans()
    return corpus.load_plan(corpus.PLAN_DIR / f"{name if name in names else name + '_ungrouped'}.plan.json")


def _grid(name, dtype, device, seed=7):
    plan = _load_plan(name)
    _, cos = corpus.lattice_of(name)
    hi = CONFIGS[name]
    grid = CoefficientGrid.zeros(cos, [0, 0, 0], [hi, hi, hi], device=device, dtype=dtype)
    gen = torch.Generator(device=device).manual_seed(seed)
    for a in grid.arrays:
        a.copy_(torch.rand(a.shape, generator=gen, device=device, dtype=torch.float32).to(dtype))
    return plan, grid, hi


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
@pytest.mark.parametrize("name", list(CONFIGS))
def test_full_size_subsample_vs_oracle(name, dtype, cuda):
    """BASELINE grid sizes, 4e6 Morton-ordered points (+ 4096 dyadic plane-tie points) through
    the brick kernels; 12,288 of them checked against the oracle (pinned to the reference):
    values within 1e-5 (fp32) / 1e-12 (fp64) of max|f| and classes + cells bit-exact."""
    from oracle.plan_numpy import classify_batch

    plan, grid, hi = _grid(name, dtype, cuda)
    n = 4_000_000
    gen = torch.Generator(device=cuda).manual_seed(3)
    pts = (torch.rand((n, 3), generator=gen, device=cuda) * (hi + 1)).to(dtype)
    ties = torch.floor(torch.rand((4096, 3), generator=gen, device=cuda) * (hi + 1) * 4) / 4  # x.0 / .25 / .5 / .75
    pts = torch.cat([pts, ties.to(dtype)])
    pts = pts[morton_order(pts)].contiguous()
    interp = PlanInterpreter(plan)
    out = interp.eval_batch(grid, pts, order="morton")
    idx = torch.cat([torch.randint(0, pts.shape[0], (8192,), generator=gen, device=cuda),
                     torch.nonzero((pts * 4 == torch.floor(pts * 4)).all(1)).flatten()[:4096]])
    sub = pts[idx].double().cpu().numpy()
    ngrid = NumpyGrid(plan.diag, plan.shifts, [a.double().cpu().numpy() for a in grid.arrays], grid.origins, "zero")
    ref = oracle_eval(plan, ngrid, sub, PlanTables(plan))
    got = out[idx].double().cpu().numpy()
    tol = 1e-5 if dtype == torch.float32 else 1e-12
    assert np.abs(got - ref).max() <= tol * np.abs(ref).max(), (name, np.abs(got - ref).max())
    cls, cells = interp.classify(grid, pts[idx])
    rcls, rcells = classify_batch(plan, sub)
    np.testing.assert_array_equal(cls.cpu().numpy(), rcls)
    np.testing.assert_array_equal(cells.cpu().numpy(), rcells)


@pytest.mark.parametrize("name", ["cc_tricubic", "bcc_linear_rd"])
def test_shift_invariance(name, cuda):
    """eval(grid shifted by D z, x + D z) == eval(grid, x) for interior x."""
    plan, grid, hi = _grid(name, torch.float64, cuda)
    gen = torch.Generator(device=cuda).manual_seed(11)
    pts = torch.rand((100_000, 3), generator=gen, device=cuda, dtype=torch.float64) * (hi - 20) + 10
    interp = PlanInterpreter(plan)
    a = interp.eval_batch(grid, pts)
    d = plan.diag[0]
    shift = (3 * d, -2 * d, 5 * d)
    moved = CoefficientGrid(grid.cosets, grid.arrays,
                            [tuple(o + s // d for o, s in zip(org, shift)) for org in grid.origins],
                            "zero", device=cuda)
    b = interp.eval_batch(moved, pts + torch.tensor(shift, dtype=torch.float64, device=cuda))
    assert (a - b).abs().max().item() <= 1e-12


def test_tricubic_fp64_full_size(cuda):
    plan, grid, hi = _grid("cc_tricubic", torch.float64, cuda)
    n = 2_000_000
    gen = torch.Generator(device=cuda).manual_seed(5)
    pts = torch.rand((n, 3), generator=gen, device=cuda, dtype=torch.float64) * (hi + 1)
    out = PlanInterpreter(plan).eval_batch(grid, pts, reorder=True)
    idx = torch.randint(0, n, (2000,), generator=gen, device=cuda)
    sub = pts[idx].cpu().numpy()
    ngrid = NumpyGrid(plan.diag, plan.shifts, [a.cpu().numpy() for a in grid.arrays], grid.origins, "zero")
    ref = oracle_eval(plan, ngrid, sub, PlanTables(plan))
    assert np.abs(out[idx].cpu().numpy() - ref).max() <= 1e-12


@pytest.mark.gpu
@pytest.mark.parametrize("name,boundary", [("bcc_quintic_rd", "zero"), ("cc_tricubic", "clamp"), ("fcc_cubic", "zero")])
def test_slab_halo_covers_the_gpu_kernels(name, boundary, cuda):
    """Slab partition (sharding.SlabPartition) with the real kernels: every rank's points
    evaluated by PlanInterpreter on that rank's slab (+ halo) views equal the evaluation on the
    whole lattice bit for bit (the routing itself is covered by the gloo tests)."""
    from paper_2102_08514_b200.runtime import CoefficientGrid, PlanInterpreter
    from paper_2102_08514_b200.sharding import SlabPartition, halo_cells

    plan = corpus.build_plan(name)
    _, cos = corpus.lattice_of(name)
    lo, hi = [0, 0, 0], [95, 31, 31]
    grid = CoefficientGrid.zeros(cos, lo, hi, boundary=boundary, device=cuda, dtype=torch.float32)
    for a in grid.arrays:
        a.copy_(torch.rand(a.shape, generator=torch.Generator(device=cuda).manual_seed(3), device=cuda))
    interp = PlanInterpreter(plan)
    gen = torch.Generator(device=cuda).manual_seed(4)
    pts = torch.rand((300_000, 3), generator=gen, device=cuda) * torch.tensor([104.0, 36.0, 36.0], device=cuda) - 4.0
    want = interp.eval_batch(grid, pts)
    world = 4
    part = SlabPartition(cos, lo, hi, world, halo_cells(plan), boundary)
    own = part.owner(pts)
    for r in range(world):
        arrays, origins = part.local_views(grid, r)
        local = CoefficientGrid(cos, [a.contiguous() for a in arrays], origins, boundary, device=cuda)
        sel = own == r
        got = interp.eval_batch(local, pts[sel])
        torch.testing.assert_close(got, want[sel], rtol=0, atol=0)


_BCC_VARIANT_SCRIPT = r"""
import sys, torch
sys.path[:0] = [sys.argv[1], sys.argv[1] + "/tests"]
from test_gpu_scale import _bcc_variant_case
name = sys.argv[4] if len(sys.argv) > 4 else "bcc_linear_rd"
torch.save(_bcc_variant_case(torch.device("cuda", 0), getattr(torch, sys.argv[3]), name), sys.argv[2])
"""


def _bcc_variant_case(cuda, dtype, name="bcc_linear_rd"):
    """A BASELINE grid: 2e6 Morton-ordered points plus points the fast loops must route to
    their checked path (outside the grid, |x| beyond the float fast domain, NaN, plane ties),
    evaluated through the brick kernels (the variant the process's environment selects)."""
    plan, grid, hi = _grid(name, dtype, cuda)
    gen = torch.Generator(device=cuda).manual_seed(21)
    pts = (torch.rand((2_000_000, 3), generator=gen, device=cuda) * (hi + 9) - 4).to(dtype)
    ties = torch.floor(torch.rand((8192, 3), generator=gen, device=cuda) * (hi + 1) * 2) / 2
    odd = torch.tensor([[float("nan"), 3.0, 4.0], [5e6, 1.0, 2.0], [-3e7, 7.5, 1.0], [1e30, 2.0, 2.0]],
                       device=cuda).repeat(64, 1)
    pts = torch.cat([pts, ties.to(dtype), odd.to(dtype)])
    pts = pts[morton_order(pts)].contiguous()
    return PlanInterpreter(plan).eval_batch(grid, pts, order="morton").cpu()


@pytest.mark.parametrize("dtype", ["float32", "float64"])
def test_bcc_linear_lean_kernel_is_bit_identical(dtype, cuda, tmp_path):
    """The default BCC linear brick kernel (bcc_tet_brick_kernel_v2: magic-number rint,
    quad-level brick test) returns the same bits as the round-2 kernel (SP_BCC_TET_VARIANT=3)
    and as the generic brick driver (BccTetEval), NaN positions included."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = {}
    for label, env in (("v2", {}), ("v1", {"SP_BCC_TET_VARIANT": "3"}), ("generic", {"SP_BCC_TET_BRICK": "0"})):
        path = str(tmp_path / f"{label}.pt")
        r = subprocess.run([sys.executable, "-c", _BCC_VARIANT_SCRIPT, root, path, dtype, "bcc_linear_rd"],
                           env=dict(os.environ, **env), capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        outs[label] = torch.load(path)
    a = outs["v2"]
    assert torch.isnan(a).sum().item() == 64
    for label in ("v1", "generic"):
        b = outs[label]
        assert torch.equal(torch.isnan(a), torch.isnan(b)), label
        assert torch.equal(a.nan_to_num(0.0).view(torch.int32 if a.dtype == torch.float32 else torch.int64),
                           b.nan_to_num(0.0).view(torch.int32 if b.dtype == torch.float32 else torch.int64)), label


@pytest.mark.parametrize("name,dtype", [("cc_tricubic", "float32"), ("cc_trilinear", "float32"),
                                        ("cc_tricubic", "float64"), ("bcc_quintic_rd", "float32"),
                                        ("cc_zp3", "float32")])
def test_plain_point_loops_are_bit_identical(name, dtype, cuda, tmp_path):
    """The plain-point loops of brick_kernel_tma / brick_kernel (direct loads and stores,
    inside-the-brick test from the floor conversions + one NaN test) return the same bits as
    the checked loops (SP_PLAIN_PTS=0) on BASELINE grids with outliers, NaN and ties."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = {}
    for label, env in (("plain", {}), ("checked", {"SP_PLAIN_PTS": "0"})):
        path = str(tmp_path / f"{label}.pt")
        r = subprocess.run([sys.executable, "-c", _BCC_VARIANT_SCRIPT, root, path, dtype, name],
                           env=dict(os.environ, **env), capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        outs[label] = torch.load(path)
    a, b = outs["plain"], outs["checked"]
    assert torch.isnan(a).sum().item() == 64
    assert torch.equal(torch.isnan(a), torch.isnan(b))
    it = torch.int32 if a.dtype == torch.float32 else torch.int64
    assert torch.equal(a.nan_to_num(0.0).view(it), b.nan_to_num(0.0).view(it))
