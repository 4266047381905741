"""CPU: the C-ABI library loads and exports every symbol include/splinerecon.h declares."""
import ctypes
import os
import re

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
