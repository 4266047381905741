"""Volume documents (runtime.py:445-494): byte parity with the reference's write_volume,
header checks, and the pinned-buffer device loader.  Fixtures: tests/golden/volume/
(made by the reference, tests/golden/make_volume_golden.py)."""
import os

import numpy as np
import pytest
import torch

from conftest import GOLDEN
from paper_2102_08514_b200 import decompose_cartesian, named_lattice
from paper_2102_08514_b200.runtime import CoefficientGrid, RuntimeError_
from paper_2102_08514_b200.volume import load_volume, parse_header, read_volume, save_volume, write_volume

VOL = os.path.join(GOLDEN, "volume")
CASES = [("CC3", "zero"), ("BCC", "mirror"), ("FCC", "clamp")]


def _fixture(lat, boundary):
    tag = f"{lat}_{boundary}"
    with np.load(os.path.join(VOL, "fixtures.npz")) as z:
        origins = [tuple(int(v) for v in o) for o in z[f"{tag}_origins"]]
        cos = decompose_cartesian(named_lattice(lat))
        arrays = [z[f"{tag}_coset{k}"] for k in range(cos.M)]
    with open(os.path.join(VOL, f"{tag}.bin"), "rb") as fh:
        data = fh.read()
    return cos, arrays, origins, data


@pytest.mark.parametrize("lat,boundary", CASES)
def test_read_and_write_match_reference_bytes(lat, boundary):
    cos, arrays, origins, data = _fixture(lat, boundary)
    g = read_volume(data, cos, device="cpu")
    assert g.boundary == boundary and g.origins == origins
    for a, b in zip(g.arrays, arrays):
        assert a.dtype == torch.float64
        np.testing.assert_array_equal(a.numpy(), b)
    assert write_volume(g) == data
    own = CoefficientGrid(cos, arrays, origins, boundary, device="cpu", dtype=torch.float64)
    assert write_volume(own) == data


def test_header_errors():
    cos, _, _, data = _fixture("BCC", "mirror")
    with pytest.raises(RuntimeError_):
        read_volume(data, decompose_cartesian(named_lattice("FCC")), device="cpu")
    with pytest.raises(RuntimeError_):
        read_volume(data, decompose_cartesian(named_lattice("CC3")), device="cpu")
    with pytest.raises(RuntimeError_):
        read_volume(b"nonsense\ndata\n", cos, device="cpu")
    fields, pos = parse_header(data)
    assert fields["lattice"] == ["BCC"] and fields["boundary"] == ["mirror"] and len(fields["extent"]) == 2
    assert pos == data.index(b"data\n") + 5


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
@pytest.mark.parametrize("lat,boundary", CASES)
def test_load_volume_to_device(lat, boundary, dtype, cuda, tmp_path):
    cos, arrays, origins, data = _fixture(lat, boundary)
    path = os.path.join(VOL, f"{lat}_{boundary}.bin")
    g = load_volume(path, cos, device=cuda, dtype=dtype)
    assert g.device.type == "cuda" and g.dtype == dtype and g.origins == origins and g.boundary == boundary
    for a, b in zip(g.arrays, arrays):
        np.testing.assert_array_equal(a.cpu().numpy(), b.astype(torch.empty(0, dtype=dtype).numpy().dtype))
    if dtype == torch.float64:
        out = tmp_path / "rt.bin"
        save_volume(str(out), g)
        assert out.read_bytes() == data
    with pytest.raises(RuntimeError_):
        trunc = tmp_path / "trunc.bin"
        trunc.write_bytes(data[:-8])
        load_volume(str(trunc), cos, device=cuda)


@pytest.mark.gpu
def test_loaded_volume_evaluates_like_direct_grid(cuda):
    """A plan evaluated on the loaded grid equals the same plan on the in-memory grid."""
    from paper_2102_08514_b200 import corpus
    from paper_2102_08514_b200.runtime import PlanInterpreter

    cos, arrays, origins, _ = _fixture("BCC", "mirror")
    plan = corpus.build_plan("bcc_linear_rd")
    g = load_volume(os.path.join(VOL, "BCC_mirror.bin"), cos, device=cuda, dtype=torch.float64)
    direct = CoefficientGrid(cos, arrays, origins, "mirror", device=cuda, dtype=torch.float64)
    pts = torch.rand((5000, 3), dtype=torch.float64, device=cuda) * 12 - 1
    interp = PlanInterpreter(plan)
    torch.testing.assert_close(interp.eval_batch(g, pts), interp.eval_batch(direct, pts), rtol=0, atol=0)
