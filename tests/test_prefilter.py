"""Quasi-interpolation prefilter on coset grids.

Pins: tests/golden/prefilter/*.npz were produced with the reference's own taps
(corpus.prefilter_taps) and policy-aware site reads (CoefficientGrid.site_value), one site
at a time (tests/golden/make_prefilter_golden.py).  The numpy oracle must reproduce them
bit for bit; the CUDA stencil (sp_prefilter) must equal them bit for bit in float64 and to
float32 rounding in float32."""
import glob
import os

import numpy as np
import pytest
import torch

from conftest import GOLDEN
from oracle.plan_numpy import NumpyGrid
from oracle.prefilter_numpy import apply_prefilter as oracle_prefilter
from oracle.prefilter_numpy import stencil_table
from paper_2102_08514_b200 import corpus, decompose_cartesian, named_lattice
from paper_2102_08514_b200.prefilter import stencil_taps

CASES = sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, "prefilter", "*.npz")))
BOUNDARIES = ("zero", "clamp", "mirror")


def _case(name):
    with np.load(os.path.join(GOLDEN, "prefilter", f"{name}.npz")) as z:
        d = {k: z[k] for k in z.files}
    cos = decompose_cartesian(named_lattice(str(d["lattice"])))
    taps = {tuple(int(v) for v in o): float(w) for o, w in zip(d["offsets"], d["taps"])}
    ins = [d[f"in{k}"] for k in range(cos.M)]
    origins = [tuple(int(v) for v in o) for o in d["origins"]]
    return d, cos, taps, ins, origins


def test_cases_present():
    assert {"bcc_quintic", "identity_cc", "shift_cc", "asym_fcc", "asym_bcc"} <= set(CASES)


@pytest.mark.parametrize("name", CASES)
@pytest.mark.parametrize("boundary", BOUNDARIES)
def test_oracle_matches_reference_loop(name, boundary):
    d, cos, taps, ins, origins = _case(name)
    g = NumpyGrid(cos.diag, cos.shifts, ins, origins, boundary)
    outs = oracle_prefilter(g, list(taps), list(taps.values()))
    for k, o in enumerate(outs):
        np.testing.assert_array_equal(o, d[f"out_{boundary}{k}"])


@pytest.mark.parametrize("name", CASES)
def test_host_stencil_resolution_matches_oracle(name):
    _, cos, taps, _, _ = _case(name)
    ours = stencil_taps(cos, taps)
    ref = stencil_table(cos.diag, cos.shifts, list(taps), list(taps.values()))
    assert ours == ref


def test_corpus_taps_match_reference_fixture():
    d, _, taps, _, _ = _case("bcc_quintic")
    mine = {o: float(w) for o, w in corpus.prefilter_taps("bcc_quintic_rd").items()}
    assert mine == taps
    assert corpus.prefilter_taps("cc_trilinear") == {(0, 0, 0): 1}
    assert sum(corpus.prefilter_taps("bcc_quintic_rd").values()) == 1  # reproduces constants


@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES)
@pytest.mark.parametrize("boundary", BOUNDARIES)
@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_gpu_prefilter_matches_reference(name, boundary, dtype, cuda):
    from paper_2102_08514_b200.prefilter import apply_prefilter
    from paper_2102_08514_b200.runtime import CoefficientGrid

    d, cos, taps, ins, origins = _case(name)
    grid = CoefficientGrid(cos, ins, origins, boundary, device=cuda, dtype=dtype)
    out = apply_prefilter(grid, taps)
    assert out.origins == grid.origins and out.boundary == boundary and out.dtype == dtype
    for k, a in enumerate(out.arrays):
        ref = d[f"out_{boundary}{k}"]
        if dtype == torch.float64:
            np.testing.assert_array_equal(a.cpu().numpy(), ref)
        else:
            scale = max(1.0, np.abs(ref).max())
            np.testing.assert_allclose(a.cpu().numpy(), ref, rtol=0, atol=2e-6 * scale)


@pytest.mark.gpu
def test_gpu_prefilter_properties_at_scale(cuda):
    """BASELINE C3 size (BCC 2x203^3): identity taps copy exactly; the quintic taps sum to
    1 (constant fields with the clamp policy stay constant); linearity."""
    from paper_2102_08514_b200.prefilter import apply_prefilter
    from paper_2102_08514_b200.runtime import CoefficientGrid, RuntimeError_

    cos = decompose_cartesian(named_lattice("BCC"))
    grid = CoefficientGrid.zeros(cos, [0, 0, 0], [405, 405, 405], "clamp", device=cuda, dtype=torch.float32)
    gen = torch.Generator(device=cuda).manual_seed(7)
    for a in grid.arrays:
        a.copy_(torch.rand(a.shape, generator=gen, device=cuda))
    ident = apply_prefilter(grid, {(0, 0, 0): 1})
    for a, b in zip(ident.arrays, grid.arrays):
        assert torch.equal(a, b)
    taps = corpus.prefilter_taps("bcc_quintic_rd")
    const = CoefficientGrid(cos, [torch.full_like(a, 0.75) for a in grid.arrays], grid.origins, "clamp",
                            device=cuda, dtype=torch.float32)
    for a in apply_prefilter(const, taps).arrays:
        torch.testing.assert_close(a, torch.full_like(a, 0.75), rtol=0, atol=1e-6)
    two = CoefficientGrid(cos, [2.5 * a + 1.0 for a in grid.arrays], grid.origins, "clamp", device=cuda,
                          dtype=torch.float32)
    pa, pb = apply_prefilter(grid, taps), apply_prefilter(two, taps)
    for a, b in zip(pa.arrays, pb.arrays):
        torch.testing.assert_close(b, 2.5 * a + 1.0, rtol=0, atol=2e-5)
    with pytest.raises(RuntimeError_):
        apply_prefilter(grid, taps, out=grid)
    with pytest.raises(RuntimeError_):
        apply_prefilter(grid, {(1, 0, 0): 1.0})  # not a BCC lattice vector


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
@pytest.mark.parametrize("boundary", ["zero", "clamp"])
@pytest.mark.parametrize("hi2", [255, 251, 253])  # coset rows of 128 (TMA / bulk), 126 (bulk), 127 (cp.async fp32)
def test_tma_and_cpasync_staging_agree_with_oracle(dtype, boundary, hi2, cuda):
    """Coset rows that are a multiple of 16 bytes with the 'zero' policy take the TMA plane
    path (zero-filled out of range), rows whose 16-byte phase repeats every two rows the
    bulk-row path, everything else element-wise cp.async; all equal the
    oracle's per-site correlation (float64: bit for bit) on a BCC grid with tiles spanning
    several z chunks and partial edge tiles."""
    import numpy as np

    from paper_2102_08514_b200.prefilter import apply_prefilter
    from paper_2102_08514_b200.runtime import CoefficientGrid

    _, cos = corpus.lattice_of("bcc_quintic_rd")
    grid = CoefficientGrid.zeros(cos, [0, 0, 0], [141, 77, hi2], boundary=boundary, device=cuda, dtype=dtype)
    rng = np.random.default_rng(12)
    for a in grid.arrays:
        a.copy_(torch.from_numpy(rng.random(tuple(a.shape))))
    taps = corpus.prefilter_taps("bcc_quintic_rd")
    got = [a.double().cpu().numpy() for a in apply_prefilter(grid, taps).arrays]
    ng = NumpyGrid(cos.diag, cos.shifts, [a.double().cpu().numpy() for a in grid.arrays], grid.origins, boundary)
    want = oracle_prefilter(ng, list(taps), [float(w) for w in taps.values()])
    for g_, w_ in zip(got, want):
        if dtype == torch.float64:
            np.testing.assert_array_equal(g_, w_)
        else:
            np.testing.assert_allclose(g_, w_, rtol=0, atol=2e-6)
