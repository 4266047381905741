"""Test/tooling-only helpers to import the read-only reference package in THIS container.

The reference (`/root/reference/pkg/src/splineplan`) falls back to `fractions` when
gmpy2 is absent, and its `rat(float)` then raises; a tiny gmpy2 shim fixes that
(SURVEY.md §8c caveat 1).  Its PP cache defaults to a path inside the read-only tree,
so SPLINEPLAN_CACHE is pointed at a writable directory (caveat 2).
Nothing in the product imports this module.
"""
import os
import sys
import tempfile

REF_SRC = "/root/reference/pkg/src"

_SHIM = '''from fractions import Fraction
def mpq(num=0, den=1):
    return Fraction(num) / Fraction(den) if den != 1 else Fraction(num)
'''


def import_reference(cache_dir: str | None = None):
    shim_dir = os.path.join(tempfile.gettempdir(), "splineplan_gmpy2_shim")
    os.makedirs(shim_dir, exist_ok=True)
    path = os.path.join(shim_dir, "gmpy2.py")
    if not os.path.exists(path):
        with open(path, "w") as fh:
            fh.write(_SHIM)
    if shim_dir not in sys.path:
        sys.path.insert(0, shim_dir)
    os.environ.setdefault("SPLINEPLAN_CACHE", cache_dir or os.path.join(tempfile.gettempdir(), "spcache"))
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    import splineplan  # noqa: F401
    return splineplan
