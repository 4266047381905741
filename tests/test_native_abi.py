"""CPU: the C-ABI library loads and exports every symbol include/splinerecon.h declares."""
import ctypes
import os
import re

import pytest

from paper_2102_08514_b200 import _native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "splinerecon.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(sp_[a-z_0-9]+)\s*\(", text)))


def test_header_symbols_exported():
    lib = ctypes.CDLL(_native.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 10
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_native.EXPORTS), "ctypes binding covers exactly the header"


def test_version_and_error_without_gpu():
    lib = _native.lib()
    assert b"sm_100a" in lib.sp_version()
    # null-argument validation does not need a device
    rc = lib.sp_plan_create(None, None)
    assert rc == _native.SP_ERR_INVALID
    assert b"null" in lib.sp_last_error()


_CHECKED_SCRIPT = r"""
import sys, ctypes, torch
from paper_2102_08514_b200 import corpus, _native
from paper_2102_08514_b200.runtime import CoefficientGrid, PlanInterpreter
assert _native.LIB_PATH.endswith("libsplinerecon_checked.so"), _native.LIB_PATH
bad = sys.argv[1] == "bad"
plan = corpus.build_plan("cc_tricubic")
_, cos = corpus.lattice_of("cc_tricubic")
dev = torch.device("cuda", 0)
grid = CoefficientGrid.zeros(cos, [0, 0, 0], [31, 31, 31], device=dev, dtype=torch.float32)
grid.arrays[0].copy_(torch.rand(grid.arrays[0].shape, device=dev))
interp = PlanInterpreter(plan)
n = 1000
pts = (torch.rand((n, 3), device=dev) * 4 + 8).contiguous()   # one brick
perm = torch.arange(n, dtype=torch.int32, device=dev)
if bad:
    perm[7] = n + 100                                         # outside the point array
start = torch.tensor([0, n], dtype=torch.int64, device=dev)
count = torch.ones(1, dtype=torch.int32, device=dev)
out = torch.empty(n, device=dev)
lib = _native.lib()
gd = grid.descriptor()
st = torch.cuda.current_stream(dev)
_native.check(lib.sp_eval_bricks_indirect(interp._handle(dev), ctypes.byref(gd), pts.data_ptr(), n,
                                          _native.SP_F32, start.data_ptr(), count.data_ptr(), 1,
                                          interp.brick_log2(grid), perm.data_ptr(), out.data_ptr(), None,
                                          st.cuda_stream))
torch.cuda.synchronize()
torch.testing.assert_close(out, interp.eval_batch(grid, pts, order="given"), rtol=0, atol=0)
print("clean")
"""


@pytest.mark.gpu
def test_checked_build_traps_on_bad_index(tmp_path):
    """The bounds-checked library (SP_CHECKED=1) evaluates a clean permuted brick exactly and
    traps — a CUDA error, not silent garbage — when the permutation points outside the
    point array (positive control for the checked-build test runs)."""
    import os
    import subprocess
    import sys

    script = tmp_path / "checked.py"
    script.write_text(_CHECKED_SCRIPT)
    env = dict(os.environ, SP_CHECKED="1", PYTHONPATH=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    ok = subprocess.run([sys.executable, str(script), "good"], env=env, capture_output=True, text=True, timeout=300)
    assert ok.returncode == 0 and "clean" in ok.stdout, ok.stdout + ok.stderr
    bad = subprocess.run([sys.executable, str(script), "bad"], env=env, capture_output=True, text=True, timeout=300)
    assert bad.returncode != 0 and "clean" not in bad.stdout, bad.stdout + bad.stderr
    assert "bounds check failed" in bad.stdout + bad.stderr or "CUDA" in bad.stdout + bad.stderr, bad.stderr[-2000:]


def test_checked_library_exports_the_same_symbols():
    """The bounds-checked build is the same ABI."""
    path = _native.LIB_PATH.replace("libsplinerecon.so", "libsplinerecon_checked.so")
    if not os.path.exists(path):
        pytest.skip("libsplinerecon_checked.so not built (build.py --checked)")
    h = ctypes.CDLL(path)
    for name in declared_symbols():
        assert hasattr(h, name), name
