"""ctypes binding of libsplinerecon.so (include/splinerecon.h).

The library is built in-tree (`python -m paper_2102_08514_b200.build`).  There is no
fallback: if the library is missing, importing the runtime's GPU entry points fails
loudly.
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

from .packing import SP_MAX_DIM, PackedPlan

SP_MAX_COSETS = 8
# SP_CHECKED=1 loads the bounds-checked build (build.py --checked) instead
LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)),
                        "libsplinerecon_checked.so" if os.environ.get("SP_CHECKED") == "1" else "libsplinerecon.so")

SP_OK = 0
SP_ERR_INVALID = -1
SP_ERR_UNSUPPORTED = -2
SP_ERR_CUDA = -3
SP_ERR_SENTINEL = -4
SP_ERR_MISMATCH = -5
SP_F32, SP_F64 = 0, 1
BOUNDARY_CODES = {"zero": 0, "clamp": 1, "mirror": 2}
KIND_NAMES = {0: "tensor_bspline", 1: "generated", 2: "generic"}

_i32p = ctypes.POINTER(ctypes.c_int32)
_f64p = ctypes.POINTER(ctypes.c_double)


class PlanDesc(ctypes.Structure):
    _fields_ = [
        ("s", ctypes.c_int32),
        ("M", ctypes.c_int32),
        ("diag", ctypes.c_int32 * SP_MAX_DIM),
        ("shifts", (ctypes.c_int32 * SP_MAX_DIM) * SP_MAX_COSETS),
        ("Q", ctypes.c_int32),
        ("normals", _i32p),
        ("offsets", _f64p),
        ("r", ctypes.c_int32),
        ("sigma", _i32p),
        ("N", ctypes.c_int32),
        ("cls_kernel", _i32p),
        ("cls_T", _f64p),
        ("cls_t", _f64p),
        ("cls_piA", _i32p),
        ("cls_pib", _i32p),
        ("K", ctypes.c_int32),
        ("kernel_group_start", _i32p),
        ("n_groups", ctypes.c_int32),
        ("group_span", _i32p),
        ("group_nspan", _i32p),
        ("group_site_start", _i32p),
        ("sites", _i32p),
        ("group_poly_start", _i32p),
        ("n_polys", ctypes.c_int32),
        ("poly_term_start", _i32p),
        ("term_exps", _i32p),
        ("term_coeffs", _f64p),
        ("texel_offset_half", ctypes.c_int32),
        ("tp_degree", ctypes.c_int32),
    ]


class GridDesc(ctypes.Structure):
    _fields_ = [
        ("s", ctypes.c_int32),
        ("M", ctypes.c_int32),
        ("dtype", ctypes.c_int32),
        ("boundary", ctypes.c_int32),
        ("diag", ctypes.c_int32 * SP_MAX_DIM),
        ("shifts", (ctypes.c_int32 * SP_MAX_DIM) * SP_MAX_COSETS),
        ("data", ctypes.c_void_p * SP_MAX_COSETS),
        ("extent", (ctypes.c_int64 * SP_MAX_DIM) * SP_MAX_COSETS),
        ("origin", (ctypes.c_int64 * SP_MAX_DIM) * SP_MAX_COSETS),
    ]


SP_MAX_STENCIL = 64


class StencilDesc(ctypes.Structure):
    """sp_stencil_desc (include/splinerecon.h)."""

    _fields_ = [
        ("M", ctypes.c_int32),
        ("tap_start", ctypes.c_int32 * (SP_MAX_COSETS + 1)),
        ("src_coset", ctypes.POINTER(ctypes.c_int32)),
        ("dz", ctypes.POINTER(ctypes.c_int32)),
        ("weight", ctypes.POINTER(ctypes.c_double)),
    ]


SP_MAX_TRANSFER = 16


class Camera(ctypes.Structure):
    """sp_camera (splinerecon.h)."""
    _fields_ = [("position", ctypes.c_double * 3), ("right", ctypes.c_double * 3), ("up", ctypes.c_double * 3),
                ("forward", ctypes.c_double * 3), ("fov", ctypes.c_double), ("step", ctypes.c_double),
                ("lattice_scale", ctypes.c_double), ("lattice_offset", ctypes.c_double * 3)]


class Transfer(ctypes.Structure):
    """sp_transfer (splinerecon.h)."""
    _fields_ = [("n", ctypes.c_int32), ("points", ctypes.c_double * (5 * SP_MAX_TRANSFER))]


EXPORTS = {
    "sp_plan_create": (ctypes.c_int, [ctypes.POINTER(PlanDesc), ctypes.POINTER(ctypes.c_void_p)]),
    "sp_plan_destroy": (None, [ctypes.c_void_p]),
    "sp_plan_kernel_kind": (ctypes.c_int, [ctypes.c_void_p]),
    "sp_plan_kernel_name": (ctypes.c_char_p, [ctypes.c_void_p]),
    "sp_eval": (
        ctypes.c_int,
        [ctypes.c_void_p, ctypes.POINTER(GridDesc), ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32,
         ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p],
    ),
    "sp_eval_sync": (
        ctypes.c_int,
        [ctypes.c_void_p, ctypes.POINTER(GridDesc), ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32,
         ctypes.c_void_p, ctypes.c_void_p],
    ),
    "sp_eval_launch_count": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64]),
    "sp_morton_keys": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p]),
    "sp_morton_keys32": (
        ctypes.c_int,
        [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
         ctypes.c_void_p, ctypes.c_void_p],
    ),
    "sp_scatter32_blocked": (
        ctypes.c_int,
        [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_int64, ctypes.c_void_p,
         ctypes.c_void_p],
    ),
    "sp_scatter32_perm_temp_bytes": (ctypes.c_int64, [ctypes.c_int64, ctypes.c_int32]),
    "sp_scatter32_perm": (
        ctypes.c_int,
        [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p,
         ctypes.c_int64, ctypes.c_void_p],
    ),
    "sp_scatter": (
        ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p]
    ),
    "sp_gather_points": (
        ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p]
    ),
    "sp_debug_stats": (ctypes.c_int, [ctypes.c_int, ctypes.c_void_p]),
    "sp_eval_bricks": (
        ctypes.c_int,
        [ctypes.c_void_p, ctypes.POINTER(GridDesc), ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p,
         ctypes.c_int32, ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p],
    ),
    "sp_brick_log2": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32]),
    "sp_brick_runs": (
        ctypes.c_int,
        [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
         ctypes.c_int64, ctypes.c_void_p],
    ),
    "sp_brick_runs_temp_bytes": (ctypes.c_int64, [ctypes.c_int64]),
    "sp_eval_bricks_dev": (
        ctypes.c_int,
        [ctypes.c_void_p, ctypes.POINTER(GridDesc), ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p,
         ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
         ctypes.c_void_p],
    ),
    "sp_texture_create": (ctypes.c_int, [ctypes.POINTER(GridDesc), ctypes.POINTER(ctypes.c_void_p)]),
    "sp_texture_destroy": (None, [ctypes.c_void_p]),
    "sp_eval_texture": (
        ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p]
    ),
    "sp_prefilter": (ctypes.c_int, [ctypes.POINTER(GridDesc), ctypes.POINTER(StencilDesc), ctypes.c_void_p, ctypes.c_void_p]),
    "sp_ray_points": (
        ctypes.c_int, [ctypes.POINTER(Camera), ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                       ctypes.c_void_p, ctypes.c_void_p]
    ),
    "sp_composite": (
        ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_int32, ctypes.POINTER(Transfer),
                       ctypes.c_void_p, ctypes.c_void_p]
    ),
    "sp_sort_points_temp_bytes": (ctypes.c_int64, [ctypes.c_int64]),
    "sp_sort_points": (
        ctypes.c_int,
        [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
         ctypes.c_int32, ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
         ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p],
    ),
    "sp_brick_runs_points_temp_bytes": (ctypes.c_int64, [ctypes.c_int64]),
    "sp_brick_runs_points": (
        ctypes.c_int,
        [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p,
         ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p],
    ),
    "sp_sort_points_payload_temp_bytes": (ctypes.c_int64, [ctypes.c_int64, ctypes.c_int32]),
    "sp_sort_points_payload": (
        ctypes.c_int,
        [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
         ctypes.c_int32, ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
         ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p],
    ),
    "sp_eval_bricks_perm32": (
        ctypes.c_int,
        [ctypes.c_void_p, ctypes.POINTER(GridDesc), ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p,
         ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
         ctypes.c_void_p],
    ),
    "sp_eval_bricks_indirect": (
        ctypes.c_int,
        [ctypes.c_void_p, ctypes.POINTER(GridDesc), ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p,
         ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
         ctypes.c_void_p],
    ),
    "sp_eval_bricks_unordered": (
        ctypes.c_int,
        [ctypes.c_void_p, ctypes.POINTER(GridDesc), ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p,
         ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
         ctypes.c_void_p],
    ),
    "sp_last_error": (ctypes.c_char_p, []),
    "sp_version": (ctypes.c_char_p, []),
}

_lib = None
_lock = threading.Lock()


class NativeError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


def lib():
    """Load the in-tree library (once).  Raises if it has not been built."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ImportError(
                    f"{LIB_PATH} is missing: build it with `python -m paper_2102_08514_b200.build"
                    f"{' --checked' if LIB_PATH.endswith('_checked.so') else ''}` "
                    "(there is no CPU fallback)"
                )
            handle = ctypes.CDLL(LIB_PATH)
            for name, (res, args) in EXPORTS.items():
                fn = getattr(handle, name)
                fn.restype = res
                fn.argtypes = args
            _lib = handle
    return _lib


def check(code: int) -> None:
    if code != SP_OK:
        raise NativeError(code, lib().sp_last_error().decode())


def _ptr(a: np.ndarray, ctype):
    return a.ctypes.data_as(ctypes.POINTER(ctype))


def make_plan_desc(p: PackedPlan, tp_degree: int = -1):
    """Build a PlanDesc; returns (desc, keepalive) — keep the arrays alive during create."""
    d = PlanDesc()
    d.s = p.s
    d.M = p.M
    for i in range(min(p.s, SP_MAX_DIM)):
        d.diag[i] = p.diag[i]
    for k in range(min(p.M, SP_MAX_COSETS)):
        for i in range(min(p.s, SP_MAX_DIM)):
            d.shifts[k][i] = p.shifts[k][i]
    keep = []

    def arr(a, dt):
        a = np.ascontiguousarray(a, dtype=dt)
        if a.size == 0:
            a = np.zeros(1, dtype=dt)
        keep.append(a)
        return _ptr(a, ctypes.c_int32 if dt == np.int32 else ctypes.c_double)

    d.Q = p.Q
    d.normals = arr(p.normals, np.int32)
    d.offsets = arr(p.offsets, np.float64)
    d.r = p.r
    d.sigma = arr(p.sigma, np.int32)
    d.N = p.N
    d.cls_kernel = arr(p.cls_kernel, np.int32)
    d.cls_T = arr(p.cls_T, np.float64)
    d.cls_t = arr(p.cls_t, np.float64)
    d.cls_piA = arr(p.cls_piA, np.int32)
    d.cls_pib = arr(p.cls_pib, np.int32)
    d.K = p.K
    d.kernel_group_start = arr(p.kernel_group_start, np.int32)
    d.n_groups = p.n_groups
    d.group_span = arr(p.group_span, np.int32)
    d.group_nspan = arr(p.group_nspan, np.int32)
    d.group_site_start = arr(p.group_site_start, np.int32)
    d.sites = arr(p.sites, np.int32)
    d.group_poly_start = arr(p.group_poly_start, np.int32)
    d.n_polys = p.n_polys
    d.poly_term_start = arr(p.poly_term_start, np.int32)
    d.term_exps = arr(p.term_exps, np.int32)
    d.term_coeffs = arr(p.term_coeffs, np.float64)
    d.texel_offset_half = p.texel_offset_half
    d.tp_degree = tp_degree
    return d, keep
