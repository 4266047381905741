"""Reconstruct / evaluate: `CoefficientGrid` + `PlanInterpreter.eval_batch` on B200.

Drop-in for the reference runtime (runtime.py:38-276): same class and method names,
argument meanings and errors, with torch tensors (CUDA) in place of numpy arrays.

* `CoefficientGrid(cosets, arrays, origins, boundary)` — per-coset C-order arrays
  (axis s-1 fastest), site D z + l_k at arrays[k][z - origins[k]] (runtime.py:38-63).
  Arrays live in HBM as contiguous float32 or float64 tensors.
* `PlanInterpreter(plan).eval_batch(grid, pts)` — Algorithm 1 over the batch
  (runtime.py:244-248 -> :363-408), executed by libsplinerecon.so (sp_eval).  numpy
  input gives numpy float64 output, as the reference does (host<->device copies
  included); CUDA tensor input gives a CUDA tensor of the grid's dtype.
* errors: `RuntimeError_` (a ValueError, runtime.py:31-32) for unknown boundary/mode,
  grid/plan mismatch (runtime.py:250-254) and the sigma sentinel (runtime.py:380-381).

Arithmetic: the compute dtype is the grid's dtype.  Coset frames and plane tests are
always float64 (bit-exact classification); weights, fetches and the
accumulation run in the compute dtype.  fp64 grids reproduce the reference to ~1e-15
relative; fp32 grids to ~1e-7 of max|f|.
"""

from __future__ import annotations

import ctypes
import os
import threading
import itertools
import math
from typing import Callable, Sequence

import numpy as np
import torch

from . import _native
from .lattice import CosetDecomposition
from .packing import pack_plan
from .plan import EvaluationPlan, deserialize_plan

_BOUNDARIES = ("zero", "clamp", "mirror")


class RuntimeError_(ValueError):
    """runtime.py:31-32."""


def _as_tensor(a, device, dtype) -> torch.Tensor:
    if isinstance(a, torch.Tensor):
        t = a
    else:
        t = torch.from_numpy(np.ascontiguousarray(np.asarray(a)))
    if dtype is None:
        dtype = t.dtype if t.dtype in (torch.float32, torch.float64) else torch.float64
    return t.to(device=device, dtype=dtype).contiguous()


def _default_device():
    return torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() else torch.device("cpu")


class CoefficientGrid:
    """Per-coset s-dimensional arrays with a boundary policy (runtime.py:38-105)."""

    def __init__(self, cosets: CosetDecomposition, arrays: Sequence, origins: Sequence[tuple],
                 boundary: str = "zero", device=None, dtype: torch.dtype | None = None):
        if boundary not in _BOUNDARIES:
            raise RuntimeError_(f"unknown boundary policy {boundary}")
        if len(arrays) != cosets.M:
            raise RuntimeError_("one array per coset required")
        device = torch.device(device) if device is not None else _default_device()
        self.cosets = cosets
        self.arrays = [_as_tensor(a, device, dtype) for a in arrays]
        if len({a.dtype for a in self.arrays}) != 1:
            raise RuntimeError_("all coset arrays must share one dtype")
        self.origins = [tuple(int(v) for v in o) for o in origins]
        self.boundary = boundary
        s = cosets.parent.s
        for a in self.arrays:
            if a.dim() != s:
                raise RuntimeError_("array rank must match the dimension")

    @staticmethod
    def zeros(cosets: CosetDecomposition, lo: Sequence, hi: Sequence, boundary: str = "zero",
              device=None, dtype: torch.dtype = torch.float64) -> "CoefficientGrid":
        """Grid covering all sites with real coordinates in [lo, hi] (runtime.py:65-78)."""
        origins, shapes = grid_extents(cosets, lo, hi)
        device = torch.device(device) if device is not None else _default_device()
        arrays = [torch.zeros(sh, dtype=dtype, device=device) for sh in shapes]
        return CoefficientGrid(cosets, arrays, origins, boundary, device=device, dtype=dtype)

    # -- properties -------------------------------------------------------------
    @property
    def dtype(self) -> torch.dtype:
        return self.arrays[0].dtype

    @property
    def device(self) -> torch.device:
        return self.arrays[0].device

    def to(self, dtype: torch.dtype | None = None, device=None) -> "CoefficientGrid":
        return CoefficientGrid(self.cosets, [a.to(device=device or a.device, dtype=dtype or a.dtype) for a in self.arrays],
                               self.origins, self.boundary, device=device or self.device, dtype=dtype or self.dtype)

    def site_count(self) -> int:
        return sum(a.numel() for a in self.arrays)

    def nbytes(self) -> int:
        return sum(a.numel() * a.element_size() for a in self.arrays)

    # -- host-side accessors (debug / setup; not the hot path) --------------------
    def fill_from(self, fn: Callable) -> None:
        """Vectorised runtime.py:80-89: fn receives an (m, s) float64 array of real site
        coordinates and returns m values (a scalar-callable is applied per site)."""
        for k, shift in enumerate(self.cosets.shifts):
            arr = self.arrays[k]
            idx = np.stack(np.meshgrid(*[np.arange(n) for n in arr.shape], indexing="ij"), -1).reshape(-1, arr.dim())
            sites = (idx + np.array(self.origins[k])) * np.array(self.cosets.diag) + np.array(shift)
            try:
                vals = np.asarray(fn(sites.astype(np.float64)), dtype=np.float64).reshape(-1)
                if vals.size != sites.shape[0]:
                    raise ValueError
            except Exception:
                vals = np.array([fn(tuple(s)) for s in sites.tolist()], dtype=np.float64)
            arr.copy_(torch.from_numpy(vals.reshape(tuple(arr.shape))).to(arr.dtype))

    def site_value(self, site: Sequence) -> float:
        ci = self.cosets.index_of(site)
        z = tuple(c - o for c, o in zip(ci.cell, self.origins[ci.coset]))
        return self._read_scalar(ci.coset, z)

    def set_site(self, site: Sequence, value: float) -> None:
        ci = self.cosets.index_of(site)
        z = tuple(c - o for c, o in zip(ci.cell, self.origins[ci.coset]))
        arr = self.arrays[ci.coset]
        if any(v < 0 or v >= n for v, n in zip(z, arr.shape)):
            raise RuntimeError_("site outside grid storage")
        arr[z] = value

    def _read_scalar(self, coset: int, z: tuple) -> float:
        """runtime.py:109-123."""
        arr = self.arrays[coset]
        idx = []
        for v, n in zip(z, arr.shape):
            v = int(v)
            if 0 <= v < n:
                idx.append(v)
                continue
            if self.boundary == "zero":
                return 0.0
            if self.boundary == "clamp":
                idx.append(min(max(v, 0), n - 1))
            else:
                idx.append(_mirror_index(v, n))
        return float(arr[tuple(idx)])

    def fetch_nearest(self, coset: int, z: Sequence[float]) -> float:
        """runtime.py:125-128: the slot nearest to coset-grid coordinate z (Python's
        round, half to even), policy-aware."""
        origin = self.origins[coset]
        return self._read_scalar(coset, tuple(int(round(v)) - o for v, o in zip(z, origin)))

    def fetch_linear(self, coset: int, u: Sequence[float], offset_half: bool = False) -> float:
        """runtime.py:130-147: multilinear interpolation of the 2^s slots around u (the
        software form of a hardware linear fetch; -0.5 first when offset_half)."""
        if offset_half:
            u = [v - 0.5 for v in u]
        origin = self.origins[coset]
        base = [math.floor(v) for v in u]
        frac = [v - b for v, b in zip(u, base)]
        total = 0.0
        for corner in itertools.product((0, 1), repeat=len(u)):
            w = 1.0
            for f, c in zip(frac, corner):
                w *= f if c else (1.0 - f)
            if w == 0.0:
                continue
            total += w * self._read_scalar(coset, tuple(b + c - o for b, c, o in zip(base, corner, origin)))
        return total

    def descriptor(self) -> _native.GridDesc:
        """sp_grid_desc of this grid (memoised on the arrays' storage, shapes and policy:
        building it costs ~10-30 us of Python, which short launches cannot hide)."""
        key = (self.boundary, tuple((a.data_ptr(), tuple(a.shape), a.dtype) for a in self.arrays),
               tuple(self.origins))
        cached = self.__dict__.get("_desc")
        if cached is not None and cached[0] == key:
            return cached[1]
        g = self._build_descriptor()
        self.__dict__["_desc"] = (key, g)
        return g

    def _build_descriptor(self) -> _native.GridDesc:
        if self.device.type != "cuda":
            raise RuntimeError_("the grid must live on a CUDA device for evaluation")
        s = self.cosets.parent.s
        g = _native.GridDesc()
        g.s = s
        g.M = self.cosets.M
        g.dtype = _native.SP_F32 if self.dtype == torch.float32 else _native.SP_F64
        g.boundary = _native.BOUNDARY_CODES[self.boundary]
        for i in range(min(s, 3)):
            g.diag[i] = self.cosets.diag[i]
        for k, sh in enumerate(self.cosets.shifts[: _native.SP_MAX_COSETS]):
            for i in range(min(s, 3)):
                g.shifts[k][i] = sh[i]
            a = self.arrays[k]
            g.data[k] = a.data_ptr()
            for i in range(min(s, 3)):
                g.extent[k][i] = a.shape[i]
                g.origin[k][i] = self.origins[k][i]
        return g


def grid_extents(cosets: CosetDecomposition, lo: Sequence, hi: Sequence):
    """Per-coset origins and shapes of CoefficientGrid.zeros (runtime.py:65-78)."""
    origins, shapes = [], []
    for shift in cosets.shifts:
        zlo = [math.ceil((lo[i] - shift[i]) / d) for i, d in enumerate(cosets.diag)]
        zhi = [math.floor((hi[i] - shift[i]) / d) for i, d in enumerate(cosets.diag)]
        origins.append(tuple(zlo))
        shapes.append(tuple(b - a + 1 for a, b in zip(zlo, zhi)))
    return origins, shapes


def _mirror_index(v: int, n: int) -> int:
    if n == 1:
        return 0
    period = 2 * n - 2
    v = abs(v) % period
    return period - v if v >= n else v


# ---------------------------------------------------------------------------
# Plan interpretation


class PlanInterpreter:
    """Evaluation of (plan, grid, x) on the GPU; mode 'float' (runtime.py:216-248).

    The plan is validated and specialised once (sp_plan_create): tensor-product
    B-spline plans run the separable kernel (proven equal, plan.py), catalog plans run
    their build-time generated kernel, anything else the generic table-driven kernel.
    """

    def __init__(self, plan, mode: str = "float", kernel: str = "auto"):
        if mode not in ("float", "exact"):
            raise RuntimeError_(f"unknown interpreter mode {mode}")
        if kernel not in ("auto", "generic"):
            raise RuntimeError_(f"unknown kernel selection {kernel}")
        if isinstance(plan, str):
            plan = deserialize_plan(plan)
        if not isinstance(plan, EvaluationPlan):
            raise RuntimeError_("plan must be an EvaluationPlan or a plan document")
        self.plan = plan
        self.mode = mode
        self._handles: dict = {}
        # guards the lazily built caches (plan handles, textures, workspaces): evaluation from
        # many threads is safe; per-call device state is per thread and stream
        self._lock = threading.RLock()
        self._tp = plan.tensor_bspline_degree()
        self._kernel = kernel
        # s = 2 plans run as their s = 3 lift (lift.py): same operations, third axis inert
        self._lift = None
        if plan.s == 2 and mode == "float":
            from .lift import lift_plan

            self._lift = PlanInterpreter(lift_plan(plan), mode, kernel)

    # -- native plan handle (one per device) ----------------------------------
    def _handle(self, device: torch.device):
        key = device.index if device.index is not None else torch.cuda.current_device()
        h = self._handles.get(key)
        if h is not None:
            return h
        with self._lock:
            return self._create_handle(key)

    def _create_handle(self, key):
        h = self._handles.get(key)
        if h is None:
            if self.plan.s != 3:
                raise NotImplementedError(
                    f"GPU evaluation is implemented for s == 3 plans (plan {self.plan.name!r} has s={self.plan.s})"
                )
            lib = _native.lib()
            # separable kernels exist for degrees 1-3; other tensor degrees take the generic kernel
            tp = -2 if self._kernel == "generic" else (self._tp if self._tp in (1, 2, 3) else -1)
            desc, keep = _native.make_plan_desc(pack_plan(self.plan), tp)
            out = ctypes.c_void_p()
            with torch.cuda.device(key):
                code = lib.sp_plan_create(ctypes.byref(desc), ctypes.byref(out))
            del keep
            if code == _native.SP_ERR_UNSUPPORTED:
                raise NotImplementedError(lib.sp_last_error().decode())
            _native.check(code)
            h = out.value
            self._handles[key] = h
        return h

    def __del__(self):
        try:
            lib = _native._lib
            if lib is not None:
                for t in self.__dict__.get("_tex", {}).values():
                    lib.sp_texture_destroy(t)
                for h in self._handles.values():
                    lib.sp_plan_destroy(h)
        except Exception:
            pass

    def brick_log2(self, grid: CoefficientGrid) -> int:
        """Recommended brick edge (log2 unit cells) for this plan and the grid's dtype."""
        if self._lift is not None:
            from .lift import lift_grid

            return self._lift.brick_log2(lift_grid(grid))
        dtype = _native.SP_F32 if grid.dtype == torch.float32 else _native.SP_F64
        return int(_native.lib().sp_brick_log2(self._handle(grid.device), dtype))

    def prepare(self, grid: CoefficientGrid, pts: torch.Tensor, *, presorted: bool = False) -> "PointBatch":
        """Brick-order a point set for repeated evaluation on this plan/grid."""
        if self._lift is not None:
            from .lift import lift_grid, lift_points

            return self._lift.prepare(lift_grid(grid), lift_points(torch.as_tensor(pts)), presorted=presorted)
        b = self.brick_log2(grid)
        if b < 0:
            raise RuntimeError_("brick mode is not applicable to this plan")
        p = pts.to(device=grid.device, dtype=grid.dtype)
        return prepare_points(p, b, presorted=presorted)

    def program(self):
        """The plan's normative scalar program (runtime.py:227-230 -> build_program,
        plancompile.py:564-699): a minilang.KernelProgram, rendered identically to the
        reference's emit_kernel; minilang.execute runs it with injected fetches (host-side
        specification aid, like the reference's; evaluation here runs on the GPU)."""
        if self.__dict__.get("_program") is None:
            from .minilang import build_program

            self._program = build_program(self.plan)
        return self._program

    def kernel_name(self, device=None) -> str:
        if self._lift is not None:
            return self._lift.kernel_name(device)
        device = torch.device(device) if device is not None else _default_device()
        return _native.lib().sp_plan_kernel_name(self._handle(device)).decode()

    def _check_grid(self, grid: CoefficientGrid) -> None:
        """runtime.py:250-254."""
        if tuple(grid.cosets.diag) != tuple(self.plan.diag) or tuple(grid.cosets.shifts) != tuple(self.plan.shifts):
            raise RuntimeError_("grid decomposition does not match the plan header")

    # -- evaluation -------------------------------------------------------------
    def eval(self, grid: CoefficientGrid, x: Sequence) -> float:
        """Single point (runtime.py:232-242), through the same GPU batch kernel."""
        self._check_grid(grid)
        if self.mode != "float":
            raise NotImplementedError("exact-debug mode is a host-only reference aid (runtime.py:279-338)")
        pts = torch.tensor([[float(v) for v in x]], dtype=grid.dtype, device=grid.device)
        return float(self.eval_batch(grid, pts)[0])

    @staticmethod
    def _on_stream(stream, dev, fn):
        """Run fn() with `stream` as the current stream (staging, allocation, launches,
        sentinel check and read-back all ordered on it).  The stream first waits for the
        caller's current stream (inputs it produced), and the caller's stream waits for it
        afterwards, with device results recorded on the caller's stream."""
        if stream is None or dev.type != "cuda":
            return fn()
        cur = torch.cuda.current_stream(dev)
        if stream == cur:
            return fn()
        stream.wait_stream(cur)
        with torch.cuda.stream(stream):
            r = fn()
        cur.wait_stream(stream)
        for t in (r if isinstance(r, tuple) else (r,)):
            if isinstance(t, torch.Tensor) and t.device.type == "cuda":
                t.record_stream(cur)
        return r

    def eval_batch(self, grid: CoefficientGrid, pts, *, out: torch.Tensor | None = None, check: bool = True,
                   order: str = "auto", reorder: bool = False, stream: torch.cuda.Stream | None = None):
        """Batch reconstruction (runtime.py:244-248).

        pts: (n, s) numpy array (-> numpy float64 result, like the reference), tensor
        (CUDA -> CUDA tensor of the grid dtype; CPU -> CPU tensor, copies included) or a
        PointBatch.  `check` synchronises and raises RuntimeError_ on a sigma-sentinel
        hit (runtime.py:380-381).  `order` says how the points are presented:
          "auto"   (default) batches of >= 2^20 points are sampled (4096 consecutive pairs)
                   and routed to "morton" when already in Morton order, "given" when
                   consecutive points are spatially coherent, else "sort"; smaller
                   batches take "given",
          "given"  any order; chunk kernel with per-chunk staging,
          "morton" already in Morton order of floor(x) (input-order protocol A): the
                   brick runs are found and the brick kernel is used,
          "sort"   Morton-sort on the GPU, brick kernel, results scattered back to the
                   caller's order (protocol B; `reorder=True` is an alias).
        All three give bit-identical values.
        """
        self._check_grid(grid)
        if self.mode != "float":
            raise RuntimeError_("batch evaluation is float-mode only")
        if stream is not None and grid.device.type == "cuda" and stream != torch.cuda.current_stream(grid.device):
            return self._on_stream(stream, grid.device, lambda: self.eval_batch(
                grid, pts, out=out, check=check, order=order, reorder=reorder, stream=None))
        if self._lift is not None:
            from .lift import lift_grid, lift_points

            if isinstance(pts, PointBatch):
                if pts.pts.shape[1] == 2:  # a brick partition of 2-D points: same runs, lifted points
                    pts = PointBatch(lift_points(pts.pts), pts.brick_start, pts.log2_brick, pts.perm,
                                     n_bricks_dev=pts.n_bricks_dev)
            else:
                if (pts.shape[-1] if hasattr(pts, "shape") else len(pts[0])) != 2:
                    raise RuntimeError_("points must have shape (n, 2)")
                pts = lift_points(pts)
            return self._lift.eval_batch(lift_grid(grid), pts, out=out, check=check, order=order, reorder=reorder,
                                         stream=stream)
        if isinstance(pts, PointBatch):
            return self._eval_bricks(grid, pts, out=out, check=check, stream=stream)
        is_numpy = not isinstance(pts, torch.Tensor)
        dev = grid.device
        if dev.type != "cuda":
            raise RuntimeError_("the grid must live on a CUDA device for evaluation")
        if is_numpy:
            pts = torch.from_numpy(np.ascontiguousarray(np.asarray(pts, dtype=np.float64)))
        on_host = pts.device.type == "cpu"
        if order not in ("auto", "given", "morton", "sort"):
            raise RuntimeError_(f"unknown point order {order!r}")
        if reorder:
            order = "sort"
        if order == "auto":
            order = choose_order(pts) if (pts.dim() == 2 and pts.shape[0] >= self.auto_order_min
                                          and self.brick_log2(grid) >= 0) else "given"
            if order == "sort" and self._taps_per_point() < self.auto_sort_min_taps:
                order = "given"  # light plans gather from L2 faster than the sort costs
        if (on_host and not is_numpy and pts.dtype == grid.dtype and pts.is_pinned() and pts.is_contiguous()
                and pts.dim() == 2 and pts.shape[1] == self.plan.s and pts.shape[0] >= 2 * self.host_chunk
                and (out is None or (out.device.type == "cpu" and out.is_pinned()))):
            return self._eval_host_pipelined(grid, pts, out, check=check, order=order, stream=stream)
        if on_host:
            # host buffers: H2D copy of the points, D2H copy of the result (pinned -> async)
            src = pts.to(dtype=grid.dtype)
            p = src.to(dev, non_blocking=src.is_pinned())
        else:
            p = pts.to(device=dev, dtype=grid.dtype).contiguous()
        if p.dim() != 2 or p.shape[1] != self.plan.s:
            raise RuntimeError_(f"points must have shape (n, {self.plan.s})")
        n = p.shape[0]
        res = out if (out is not None and out.device == dev) else torch.empty(n, dtype=grid.dtype, device=dev)
        if n:
            self._launch(grid, p, res, check=check, order=order, stream=stream)
        if is_numpy:
            return res.to("cpu").numpy().astype(np.float64)
        if on_host:
            if out is not None and out.device.type == "cpu":
                out.copy_(res, non_blocking=out.is_pinned())
                return out
            return res.to("cpu")
        return res

    # batches at least this large are sampled by order="auto" (see choose_order)
    auto_order_min = 1 << 20

    # order="auto" sorts incoherent batches only for plans reading at least this many
    # coefficients per point: measured on B200 with 1e8 iid points, unstaged L2 gathers cost
    # ~0.9 ms per tap (tricubic 64 taps: 60 ms; BCC quintic 32: 24 ms; BCC linear 4: 4.4 ms)
    # against ~10 ms for the sort + permuted reads + scatter of protocol B
    auto_sort_min_taps = 12

    # protocol B: gather the sorted points into a contiguous copy before the brick kernel
    # (True) or let the brick kernel read them through the permutation (False)
    sort_gather = os.environ.get("SP_SORT_GATHER", "0") == "1"

    # protocol B: move the points through the radix sort as its payload (brick-id keys, the
    # points read once, coalesced) instead of reading them through the permutation.  Measured
    # (1e8 tricubic points, tools/protocol_b_timing.py): the 16-byte payload makes each onesweep
    # pass 1.1 ms (3.3 ms for 3 passes, 4.7 ms with keys and split) and brick-sorted points
    # without Morton order inside the brick cost the TMA kernel 1.97 ms instead of 0.9 — 9.14 ms
    # in total vs 9.24 ms for the permuted-read path, so it stays off by default
    sort_payload = os.environ.get("SP_SORT_PAYLOAD", "0") == "1"

    # protocol B result scatter: destination window (elements) of the L2-blocked scatter
    # (sp_scatter32_blocked); 0 = the brick kernel scatters directly (sp_eval_bricks_indirect)
    scatter_window = int(os.environ.get("SP_SCATTER_WINDOW", str(1 << 24)))
    # ... done as a radix sort of the (destination, value) pairs by the destination's high bits
    # plus one full-store pass per 2048-value window (sp_scatter32_perm) instead of one pass
    # over all pairs per L2 window
    scatter_sorted = os.environ.get("SP_SCATTER_SORTED", "1") == "1"

    # protocol-B workspaces kept (one per thread x stream x batch shape, most recent first out)
    sort_ws_keep = 4

    def _taps_per_point(self) -> float:
        counts = self.plan.nearest_fetch_counts
        counts = counts() if callable(counts) else counts
        return sum(counts) / max(1, len(counts))  # per point, over all cosets (plancompile.py:129-140)

    # points per pipelined host chunk (pinned host buffers, see _eval_host_pipelined)
    host_chunk = 1 << 22

    # device slots of the pinned-host pipeline (ring of chunk buffers)
    host_slots = 3

    def _pipeline_state(self, dev, dtype, s):
        """Per (thread, device, dtype) pipeline resources, created once: three streams (H2D
        copy, compute, D2H copy) and a ring of `host_slots` chunk buffers with their events
        (per thread, so concurrent callers never share a ring)."""
        key = (threading.get_ident(), dev, dtype, s, self.host_chunk, self.host_slots)
        with self._lock:
            st = self.__dict__.setdefault("_pipes", {}).get(key)
        if st is None:
            C = self.host_chunk
            slots = []
            for _ in range(self.host_slots):
                slots.append({
                    "p": torch.empty((C, s), dtype=dtype, device=dev),
                    "r": torch.empty(C, dtype=dtype, device=dev),
                    "scratch": torch.empty(max(1, int(_native.lib().sp_brick_runs_temp_bytes(C))), dtype=torch.uint8,
                                           device=dev),
                    "evaluated": None, "returned": None,
                })
            st = {"h2d": torch.cuda.Stream(dev), "comp": torch.cuda.Stream(dev), "d2h": torch.cuda.Stream(dev),
                  "slots": slots}
            with self._lock:
                self._pipes[key] = st
        return st

    def _eval_host_pipelined(self, grid, pts, out, *, check, order, stream):
        """Pinned host points -> pinned host results, overlapping the PCIe transfers with
        each other and with the evaluation: the batch is cut into chunks of `host_chunk`
        points that cycle through a ring of `host_slots` device buffers; chunk i is copied
        in on the H2D stream (once its slot's previous chunk is evaluated), evaluated on the
        compute stream (sync-free brick runs, no host round trip) and copied back on the D2H
        stream, so result copies overlap point copies.  Chunks are contiguous ranges, so a
        Morton-ordered batch gives Morton-ordered chunks; values are identical to the
        one-shot path (every point is evaluated by the same arithmetic)."""
        dev = grid.device
        n, s = pts.shape
        caller = stream if stream is not None else torch.cuda.current_stream(dev)
        state = self._pipeline_state(dev, grid.dtype, s)
        h2d, comp, d2h = state["h2d"], state["comp"], state["d2h"]
        res_host = out if out is not None else torch.empty(n, dtype=grid.dtype, pin_memory=True)
        for s_ in (h2d, d2h, comp):
            s_.wait_stream(caller)
        err = torch.zeros(1, dtype=torch.int32, device=dev) if check else None
        C = self.host_chunk
        slots = state["slots"]
        for i, a in enumerate(range(0, n, C)):
            b = min(a + C, n)
            m = b - a
            sl = slots[i % len(slots)]
            if sl["evaluated"] is not None:
                h2d.wait_event(sl["evaluated"])  # input slot free
            with torch.cuda.stream(h2d):
                sl["p"][:m].copy_(pts[a:b], non_blocking=True)
            copied = torch.cuda.Event()
            copied.record(h2d)
            comp.wait_event(copied)
            if sl["returned"] is not None:
                comp.wait_event(sl["returned"])  # output slot free
            self._launch(grid, sl["p"][:m], sl["r"][:m], check=False, order=order, stream=comp, err=err,
                         sync_free=True, scratch=sl["scratch"])
            ev = torch.cuda.Event()
            ev.record(comp)
            sl["evaluated"] = ev
            d2h.wait_event(ev)
            with torch.cuda.stream(d2h):
                res_host[a:b].copy_(sl["r"][:m], non_blocking=True)
            ret = torch.cuda.Event()
            ret.record(d2h)
            sl["returned"] = ret
        caller.wait_stream(d2h)
        caller.wait_stream(comp)
        if check:
            caller.synchronize()
            if int(err.item()):
                raise RuntimeError_("sigma sentinel hit in batch evaluation")
        return res_host

    def _eval_bricks(self, grid, batch: "PointBatch", *, out=None, check=True, stream=None, unpermute=True,
                     err=None):
        """Brick-mode evaluation (sp_eval_bricks).  Results are returned in the caller's
        original order (batch.perm scatter fused into the kernel) unless unpermute=False."""
        lib = _native.lib()
        dev = grid.device
        if batch.pts.device != dev or batch.pts.dtype != grid.dtype:
            raise RuntimeError_("batch points must be on the grid's device with the grid's dtype")
        h = self._handle(dev)
        gdesc = grid.descriptor()
        dtype = _native.SP_F32 if grid.dtype == torch.float32 else _native.SP_F64
        n = batch.n
        res = out if out is not None else torch.empty(n, dtype=grid.dtype, device=dev)
        st = stream if stream is not None else torch.cuda.current_stream(dev)
        if check:
            err = torch.zeros(1, dtype=torch.int32, device=dev)
        idx = batch.perm if (unpermute and batch.perm is not None) else None
        if n and batch.n_bricks_dev is not None:
            with torch.cuda.stream(st):
                _native.check(lib.sp_eval_bricks_dev(h, ctypes.byref(gdesc), batch.pts.data_ptr(), n, dtype,
                                                     batch.brick_start.data_ptr(), batch.n_bricks_dev.data_ptr(),
                                                     batch.n_bricks_cap, batch.log2_brick,
                                                     None if idx is None else idx.data_ptr(), res.data_ptr(),
                                                     None if err is None else err.data_ptr(), st.cuda_stream))
        elif n:
            with torch.cuda.stream(st):
                _native.check(lib.sp_eval_bricks(h, ctypes.byref(gdesc), batch.pts.data_ptr(), n, dtype,
                                                 batch.brick_start.data_ptr(), batch.n_bricks, batch.log2_brick,
                                                 None if idx is None else idx.data_ptr(), res.data_ptr(),
                                                 None if err is None else err.data_ptr(), st.cuda_stream))
        if check and int(err.item()):
            raise RuntimeError_("sigma sentinel hit in batch evaluation")
        return res

    def graph(self, grid: CoefficientGrid, pts, *, out: torch.Tensor):
        """One eval_batch (a PointBatch, or device points in the given order) captured in a
        CUDA graph — `graph(...).replay()` re-evaluates the same buffers with one graph launch,
        which removes the host-side cost of the call for launch-bound batches (≲ 10^7
        points).  No sigma-sentinel check inside the graph (use eval_batch for that)."""
        order = None if isinstance(pts, PointBatch) else "given"
        kw = {} if order is None else {"order": order}
        dev = grid.device
        side = torch.cuda.Stream(device=dev)
        side.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(side):  # warm-up outside capture: handles, tensor maps, occupancy caches
            self.eval_batch(grid, pts, out=out, check=False, **kw)
        torch.cuda.current_stream(dev).wait_stream(side)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self.eval_batch(grid, pts, out=out, check=False, **kw)
        return g

    def eval_batch_unordered(self, grid: CoefficientGrid, pts: torch.Tensor, *, check: bool = True,
                             stream: torch.cuda.Stream | None = None):
        """Protocol B without the return to caller order: (values, perm) with values[k] the
        reconstruction at pts[perm[k]] (perm int32 on the grid's device — a valid index tensor,
        int64 from 2^31 points; brick order: grouped by brick, caller order within a brick),
        bit-identical to eval_batch(grid, pts)[perm].  For reductions over the batch (error
        norms, sums, histograms) the random per-value result writes of eval_batch(order=
        "sort") are skipped (sp_eval_bricks_unordered).  Device points, 3-D plans."""
        self._check_grid(grid)
        if self._lift is not None or self.plan.s != 3:
            raise NotImplementedError("eval_batch_unordered: 3-D plans only")
        if stream is not None and stream != torch.cuda.current_stream(grid.device):
            return self._on_stream(stream, grid.device,
                                   lambda: self.eval_batch_unordered(grid, pts, check=check, stream=None))
        if not isinstance(pts, torch.Tensor) or pts.device != grid.device or pts.dim() != 2 or pts.shape[1] != 3:
            raise RuntimeError_("points must be an (n, 3) tensor on the grid's device")
        p = pts.to(dtype=grid.dtype).contiguous()
        n = p.shape[0]
        st = stream if stream is not None else torch.cuda.current_stream(grid.device)
        b = self.brick_log2(grid)
        frame = _sort_frame(grid, b) if b >= 0 else None
        if frame is None or not 0 < n < (1 << 31):  # no brick mode / wide grid: caller order
            with torch.cuda.stream(st):
                perm = torch.arange(n, dtype=torch.int32 if n < (1 << 31) else torch.int64, device=grid.device)
            return self.eval_batch(grid, p, check=check, order="given", stream=st), perm
        err = torch.zeros(1, dtype=torch.int32, device=grid.device) if check else None
        with torch.cuda.stream(st):
            res = torch.empty(n, dtype=grid.dtype, device=grid.device)
        perm = self._eval_sorted32(grid, p, res, b, frame, st, err, unordered=True)
        if check:
            st.synchronize()
            if int(err.item()):
                raise RuntimeError_("sigma sentinel hit in batch evaluation")
        return res, perm

    def _eval_sorted32(self, grid, p, res, b, frame, st, err, unordered=False):
        """Protocol B without host round trips: sp_sort_points (30-bit Morton keys in the
        grid's frame, CUB pair sort, brick runs) then sp_eval_bricks_indirect (the brick
        kernel reads the caller's points through the permutation and scatters the results
        back to the caller's order); sort_gather = True gathers a sorted copy first and uses
        sp_eval_bricks_perm32."""
        lib = _native.lib()
        dev = grid.device
        n = p.shape[0]
        dtype = _native.SP_F32 if grid.dtype == torch.float32 else _native.SP_F64
        (lo0, lo1, lo2), bits = frame
        # one cached workspace per (thread, stream): reuse is stream-ordered, and concurrent
        # callers never share one; allocated on `st` so that the caching
        # allocator recycles it in that stream's order when it is dropped
        payload = self.sort_payload
        key = (threading.get_ident(), st.cuda_stream, dev.index, n, grid.dtype, self.sort_gather, payload)
        with self._lock:
            cache = self.__dict__.setdefault("_sort_ws", {})
            ws = cache.pop(key, None)
        if ws is None:
            tb = (lib.sp_sort_points_payload_temp_bytes(n, dtype) if payload else lib.sp_sort_points_temp_bytes(n))
            with torch.cuda.stream(st):
                ws = (torch.empty_like(p) if (self.sort_gather or payload) else None,
                      torch.empty(n, dtype=torch.int32, device=dev),
                      torch.empty(n + 1, dtype=torch.int64, device=dev), torch.empty(1, dtype=torch.int32, device=dev),
                      torch.empty(max(1, int(tb)), dtype=torch.uint8, device=dev))
        with self._lock:
            cache[key] = ws
            while len(cache) > self.sort_ws_keep:
                cache.pop(next(iter(cache)))
        sp_, perm, start, count, tmp = ws
        h = self._handle(dev)
        gdesc = grid.descriptor()
        gather = self.sort_gather
        with torch.cuda.stream(st):
            if unordered:  # the permutation is returned: not the cached workspace's
                perm = torch.empty(n, dtype=torch.int32, device=dev)
                gather = False
            if payload:
                # points moved through the radix sort (read once, coalesced), then the brick
                # kernel on the sorted copy: results scattered to the caller's order (perm32)
                # or left in brick order (unordered)
                _native.check(lib.sp_sort_points_payload(p.data_ptr(), n, dtype, lo0, lo1, lo2, bits, b, sp_.data_ptr(),
                                                         perm.data_ptr(), start.data_ptr(), count.data_ptr(),
                                                         tmp.data_ptr(), tmp.numel(), st.cuda_stream))
                if unordered:
                    _native.check(lib.sp_eval_bricks_dev(h, ctypes.byref(gdesc), sp_.data_ptr(), n, dtype,
                                                         start.data_ptr(), count.data_ptr(), n, b, None, res.data_ptr(),
                                                         None if err is None else err.data_ptr(), st.cuda_stream))
                    return perm
                _native.check(lib.sp_eval_bricks_perm32(h, ctypes.byref(gdesc), sp_.data_ptr(), n, dtype,
                                                        start.data_ptr(), count.data_ptr(), n, b, perm.data_ptr(),
                                                        res.data_ptr(), None if err is None else err.data_ptr(),
                                                        st.cuda_stream))
                return None
            _native.check(lib.sp_sort_points(p.data_ptr(), n, dtype, lo0, lo1, lo2, bits, b,
                                             sp_.data_ptr() if gather else None, perm.data_ptr(), start.data_ptr(),
                                             count.data_ptr(), tmp.data_ptr(), tmp.numel(), st.cuda_stream))
            if unordered:
                _native.check(lib.sp_eval_bricks_unordered(h, ctypes.byref(gdesc), p.data_ptr(), n, dtype,
                                                           start.data_ptr(), count.data_ptr(), n, b, perm.data_ptr(),
                                                           res.data_ptr(), None if err is None else err.data_ptr(),
                                                           st.cuda_stream))
                return perm
            if not gather and self.scatter_window > 0 and n > self.scatter_window:
                # values in brick order, then an L2-blocked scatter to the caller's order (one
                # pass per L2-sized destination window: tools/scatter_probe.py, 1e8 values 3.8 ->
                # 2.2 ms) instead of the kernel's random 4-byte writes
                vals = torch.empty_like(res)
                _native.check(lib.sp_eval_bricks_unordered(h, ctypes.byref(gdesc), p.data_ptr(), n, dtype,
                                                           start.data_ptr(), count.data_ptr(), n, b, perm.data_ptr(),
                                                           vals.data_ptr(), None if err is None else err.data_ptr(),
                                                           st.cuda_stream))
                if self.scatter_sorted:
                    tmp2 = torch.empty(max(1, int(lib.sp_scatter32_perm_temp_bytes(n, dtype))), dtype=torch.uint8,
                                       device=dev)
                    _native.check(lib.sp_scatter32_perm(vals.data_ptr(), perm.data_ptr(), n, dtype, res.data_ptr(),
                                                        tmp2.data_ptr(), tmp2.numel(), st.cuda_stream))
                else:
                    _native.check(lib.sp_scatter32_blocked(vals.data_ptr(), perm.data_ptr(), n, dtype,
                                                           self.scatter_window, res.data_ptr(), st.cuda_stream))
                return None
            fn = lib.sp_eval_bricks_perm32 if gather else lib.sp_eval_bricks_indirect
            _native.check(fn(h, ctypes.byref(gdesc), (sp_ if gather else p).data_ptr(), n, dtype, start.data_ptr(),
                             count.data_ptr(), n, b, perm.data_ptr(), res.data_ptr(),
                             None if err is None else err.data_ptr(), st.cuda_stream))

    def eval_batch_texture(self, grid: CoefficientGrid, pts: torch.Tensor, *, out: torch.Tensor | None = None,
                           stream: torch.cuda.Stream | None = None) -> torch.Tensor:
        """Hardware-texture-filtered variant (sp_eval_texture): the paper's GPU fetch path with
        9-bit texture filtering weights — NOT within the exact tolerances; reported
        separately with its measured error.  fp32 grids, 'zero' / 'clamp' policies;
        tensor-product plans of degree 1 or 3 (8 filtered fetches per tricubic point) and the
        compiled box-spline plans (one filtered fetch per 2-site fetch group, TexFetch)."""
        self._check_grid(grid)
        if stream is not None and stream != torch.cuda.current_stream(grid.device):
            return self._on_stream(stream, grid.device,
                                   lambda: self.eval_batch_texture(grid, pts, out=out, stream=None))
        lib = _native.lib()
        h = self._handle(grid.device)
        # the texture is a snapshot of the arrays: the key includes their version counters
        # (in-place updates invalidate it), shapes, origins and the boundary policy
        key = (id(grid), tuple((a.data_ptr(), tuple(a.shape), a._version) for a in grid.arrays),
               tuple(map(tuple, grid.origins)), grid.boundary)
        with self._lock:
            tex = self._texture_for(grid, key, lib)
        p = pts.to(device=grid.device, dtype=torch.float32).contiguous()
        res = out if out is not None else torch.empty(p.shape[0], dtype=torch.float32, device=grid.device)
        st = stream if stream is not None else torch.cuda.current_stream(grid.device)
        code = lib.sp_eval_texture(h, tex, p.data_ptr(), p.shape[0], res.data_ptr(), st.cuda_stream)
        if code == _native.SP_ERR_UNSUPPORTED:
            raise NotImplementedError(lib.sp_last_error().decode())
        _native.check(code)
        return res

    def _texture_for(self, grid, key, lib):
        """The texture objects of `grid` (up to 4 grids cached; an evicted one is destroyed
        after a device synchronisation, since another thread's launch may still read it;
        caller holds the lock)."""
        cache = self.__dict__.setdefault("_tex", {})
        tex = cache.get(key)
        if tex is None:
            if len(cache) >= 4:
                torch.cuda.synchronize(grid.device)
                lib.sp_texture_destroy(cache.pop(next(iter(cache))))
            gd = grid.descriptor()
            hnd = ctypes.c_void_p()
            code = lib.sp_texture_create(ctypes.byref(gd), ctypes.byref(hnd))
            if code == _native.SP_ERR_UNSUPPORTED:
                raise NotImplementedError(lib.sp_last_error().decode())
            _native.check(code)
            tex = cache[key] = hnd.value
        return tex

    def classify(self, grid: CoefficientGrid, pts: torch.Tensor):
        """Per point and coset: class id and coset cell kk/d (runtime.py:371-379), as
        computed by the evaluation kernel itself.  Returns (classes (n,M), cells (n,M,s))."""
        self._check_grid(grid)
        if self._lift is not None:
            from .lift import lift_grid, lift_points

            cls, cells = self._lift.classify(lift_grid(grid), lift_points(torch.as_tensor(pts)))
            return cls, cells[:, :, :2]
        p = torch.as_tensor(pts).to(device=grid.device, dtype=grid.dtype).contiguous()
        n = p.shape[0]
        M = self.plan.M
        dbg = torch.empty((n, M, 4), dtype=torch.int32, device=grid.device)
        res = torch.empty(n, dtype=grid.dtype, device=grid.device)
        if n:
            self._launch(grid, p, res, dbg=dbg, check=False)
        return dbg[:, :, 0].to(torch.int64), dbg[:, :, 1:].to(torch.int64)

    def _launch(self, grid, p, res, *, dbg=None, check=True, order="given", stream=None, err=None, sync_free=False,
                scratch=None):
        """Evaluate device points p into res on `stream`.  `err` (optional int32 device flag)
        accumulates sigma-sentinel hits without synchronising; with check=True a fresh flag
        is used and tested."""
        lib = _native.lib()
        h = self._handle(grid.device)
        gdesc = grid.descriptor()
        dtype = _native.SP_F32 if grid.dtype == torch.float32 else _native.SP_F64
        st = stream if stream is not None else torch.cuda.current_stream(grid.device)
        if check:
            err = torch.zeros(1, dtype=torch.int32, device=grid.device)
        n = p.shape[0]
        b = self.brick_log2(grid) if (order != "given" and dbg is None) else -1
        if b >= 0 and order == "sort":
            frame = _sort_frame(grid, b)
            if frame is not None and 0 < n < (1 << 31):
                self._eval_sorted32(grid, p, res, b, frame, st, err)
                if check and int(err.item()):
                    raise RuntimeError_("sigma sentinel hit in batch evaluation")
                return
        if b >= 0:
            # Morton-ordered input: brick runs found on the device with the count kept there
            # (sp_brick_runs), no host round trip (prepare_points syncs for its run count)
            if sync_free or (order == "morton" and 0 < n < (1 << 31)):
                batch = prepare_points_async(p, b, presorted=(order == "morton"), stream=st, scratch=scratch)
            else:
                batch = prepare_points(p, b, presorted=(order == "morton"), stream=st)
            self._eval_bricks(grid, batch, out=res, check=check, stream=st, err=err)
            return
        with torch.cuda.stream(st):
            if order == "sort":
                perm = morton_order(p, stream=st)
                ps = torch.empty_like(p)
                _native.check(lib.sp_gather_points(p.data_ptr(), perm.data_ptr(), n, dtype, ps.data_ptr(), st.cuda_stream))
                tmp = torch.empty_like(res)
                _native.check(lib.sp_eval(h, ctypes.byref(gdesc), ps.data_ptr(), n, dtype, tmp.data_ptr(),
                                          None if dbg is None else dbg.data_ptr(),
                                          None if err is None else err.data_ptr(), st.cuda_stream))
                _native.check(lib.sp_scatter(tmp.data_ptr(), perm.data_ptr(), n, dtype, res.data_ptr(), st.cuda_stream))
            else:
                _native.check(lib.sp_eval(h, ctypes.byref(gdesc), p.data_ptr(), n, dtype, res.data_ptr(),
                                          None if dbg is None else dbg.data_ptr(),
                                          None if err is None else err.data_ptr(), st.cuda_stream))
        if check and int(err.item()):
            raise RuntimeError_("sigma sentinel hit in batch evaluation")


def _morton64(cells: np.ndarray) -> np.ndarray:
    """Morton keys (axis 2 lowest) of int64 cells biased into [0, 2^21), as sp_morton_keys."""
    c = np.clip(cells + (1 << 20), 0, (1 << 21) - 1).astype(np.uint64)
    key = np.zeros(c.shape[0], dtype=np.uint64)
    for bit in range(21):
        for axis, shift in ((2, 0), (1, 1), (0, 2)):
            key |= ((c[:, axis] >> np.uint64(bit)) & np.uint64(1)) << np.uint64(3 * bit + shift)
    return key


def choose_order(pts: torch.Tensor, pairs: int = 4096) -> str:
    """Input-order heuristic of eval_batch(order="auto") from `pairs` evenly spaced pairs
    of consecutive points: "morton" if >= 99.9 % of them are non-decreasing in Morton order
    of their unit cells (protocol A layout), "given" if the median Chebyshev jump between
    consecutive cells is <= 2 (coherent input, e.g. rays or raster scans: chunk staging
    works), else "sort" (protocol B).  On a CUDA tensor the statistics are computed on the
    device (sp_morton_keys) and two numbers cross to the host; no effect on values."""
    n = pts.shape[0]
    if n < 2:
        return "given"
    m = min(pairs, n - 1)
    # evenly spaced in int64 (a float32 linspace rounds n - 2 up to n for n ~ 1e8)
    idx = torch.arange(m, device=pts.device, dtype=torch.int64) * (n - 2) // max(m - 1, 1)
    ab = torch.cat([pts[idx], pts[idx + 1]], 0).to(torch.float64)
    ab = torch.nan_to_num(ab, nan=0.0, posinf=2.0**30, neginf=-2.0**30).clamp(-2.0**30, 2.0**30)
    cells = torch.floor(ab)
    jump = (cells[m:] - cells[:m]).abs().amax(1)
    if pts.device.type == "cuda":
        keys = torch.empty(2 * m, dtype=torch.int64, device=pts.device)
        _native.check(_native.lib().sp_morton_keys(ab.contiguous().data_ptr(), 2 * m, _native.SP_F64, keys.data_ptr(),
                                                   torch.cuda.current_stream(pts.device).cuda_stream))
        frac, med = torch.stack([(keys[m:] >= keys[:m]).double().mean(), jump.median()]).tolist()
    else:
        c = cells.numpy().astype(np.int64)
        ka, kb = _morton64(c[:m]), _morton64(c[m:])
        frac, med = float(np.mean(kb >= ka)), float(jump.median())
    if frac >= 0.999:
        return "morton"
    return "given" if med <= 2 else "sort"


def _sort_frame(grid: CoefficientGrid, log2_brick: int):
    """(lo (3 ints, brick-aligned), bits) of a 30-bit Morton frame covering the grid's unit
    cells plus a margin of 8 cells, or None when the grid needs more than 2^10 cells per axis
    (protocol B then sorts 64-bit keys).  Host-only (grid metadata): no device sync."""
    diag, shifts = grid.cosets.diag, grid.cosets.shifts
    lo, hi = [], []
    for i in range(3):
        a = min(diag[i] * grid.origins[k][i] + shifts[k][i] for k in range(len(shifts)))
        z = max(diag[i] * (grid.origins[k][i] + grid.arrays[k].shape[i] - 1) + shifts[k][i] for k in range(len(shifts)))
        lo.append(((a - 8) >> log2_brick) << log2_brick)
        hi.append(z + 8)
    bits = max(log2_brick, max(h - l for h, l in zip(hi, lo)).bit_length())
    return (tuple(lo), bits) if bits <= 10 else None


def eval_plan(interp: PlanInterpreter, grid: CoefficientGrid, x: Sequence) -> float:
    """runtime.py:275-276."""
    return interp.eval(grid, x)


class PointBatch:
    """Query points in brick order: the input layout of the brick-mode kernel.

    `pts` are sorted by the Morton code of their unit cell floor(x), so points of each
    aligned brick of (2^log2_brick)^3 unit cells are contiguous; `brick_start[b]` ..
    `brick_start[b+1]` is brick b's run.  `perm[i]` is the caller's index of sorted point i
    (None when the points were already presented in this order).  Build one with
    `prepare_points`; evaluate with `PlanInterpreter.eval_batch(grid, batch)`.
    """

    def __init__(self, pts: torch.Tensor, brick_start: torch.Tensor, log2_brick: int, perm: torch.Tensor | None,
                 n_bricks_dev: torch.Tensor | None = None):
        self.pts = pts
        self.brick_start = brick_start
        self.log2_brick = int(log2_brick)
        self.perm = perm
        # sync-free runs: the count lives on the device (int32 [1]); brick_start has
        # capacity n + 1 and only its first count + 1 entries are meaningful
        self.n_bricks_dev = n_bricks_dev

    @property
    def n(self) -> int:
        return self.pts.shape[0]

    @property
    def n_bricks(self) -> int:
        if self.n_bricks_dev is not None:
            return int(self.n_bricks_dev.item())  # synchronises
        return self.brick_start.shape[0] - 1

    @property
    def n_bricks_cap(self) -> int:
        return self.brick_start.shape[0] - 1


def prepare_points_async(pts: torch.Tensor, log2_brick: int, *, presorted: bool = False,
                         stream: torch.cuda.Stream | None = None, scratch: torch.Tensor | None = None) -> PointBatch:
    """prepare_points without any host synchronisation (64-bit Morton keys, GPU sort when
    not presorted, brick runs by sp_brick_runs with the count kept on the device), so a host
    pipeline can queue many batches back to back."""
    lib = _native.lib()
    st = stream if stream is not None else torch.cuda.current_stream(pts.device)
    pts = pts.contiguous()
    n = pts.shape[0]
    dtype = _native.SP_F32 if pts.dtype == torch.float32 else _native.SP_F64
    with torch.cuda.stream(st):
        if presorted and n:
            # brick runs straight from the points (no 8-byte key per point written and re-read)
            start = torch.empty(n + 1, dtype=torch.int64, device=pts.device)
            count = torch.empty(1, dtype=torch.int32, device=pts.device)
            need = int(lib.sp_brick_runs_points_temp_bytes(n))
            if scratch is None or scratch.numel() < need:
                scratch = torch.empty(max(need, 1), dtype=torch.uint8, device=pts.device)
            _native.check(lib.sp_brick_runs_points(pts.data_ptr(), n, dtype, int(log2_brick), start.data_ptr(),
                                                   count.data_ptr(), scratch.data_ptr(), scratch.numel(),
                                                   st.cuda_stream))
            return PointBatch(pts, start, log2_brick, None, n_bricks_dev=count)
        keys = torch.empty(n, dtype=torch.int64, device=pts.device)
        _native.check(lib.sp_morton_keys(pts.data_ptr(), n, dtype, keys.data_ptr(), st.cuda_stream))
        perm = None
        if not presorted and n:
            keys, perm = torch.sort(keys)
            sp = torch.empty_like(pts)
            _native.check(lib.sp_gather_points(pts.data_ptr(), perm.data_ptr(), n, dtype, sp.data_ptr(), st.cuda_stream))
            pts = sp
        start = torch.empty(n + 1, dtype=torch.int64, device=pts.device)
        count = torch.empty(1, dtype=torch.int32, device=pts.device)
        need = int(lib.sp_brick_runs_temp_bytes(n))
        if scratch is None or scratch.numel() < need:
            scratch = torch.empty(max(need, 1), dtype=torch.uint8, device=pts.device)
        _native.check(lib.sp_brick_runs(keys.data_ptr(), n, int(log2_brick), start.data_ptr(), count.data_ptr(),
                                        scratch.data_ptr(), scratch.numel(), st.cuda_stream))
    return PointBatch(pts, start, log2_brick, perm, n_bricks_dev=count)


def prepare_points(pts: torch.Tensor, log2_brick: int, *, presorted: bool = False,
                   stream: torch.cuda.Stream | None = None) -> PointBatch:
    """Morton-sort points (GPU) and delimit their bricks.  With presorted=True the points
    are taken to be in Morton order already (input-order protocol A) and only the brick
    runs are found."""
    lib = _native.lib()
    st = stream if stream is not None else torch.cuda.current_stream(pts.device)
    pts = pts.contiguous()
    n = pts.shape[0]
    dtype = _native.SP_F32 if pts.dtype == torch.float32 else _native.SP_F64
    with torch.cuda.stream(st):
        perm = None
        keys = None
        if not presorted and n:
            # 32-bit keys relative to the brick-aligned bounding box when it is small enough
            # (half the radix-sort width of the 64-bit keys); same order, same brick runs
            lo = pts.amin(0).floor()  # floor is monotone: min(floor(x)) = floor(min(x))
            hi = pts.amax(0).floor()
            if bool(torch.isfinite(lo).all() and torch.isfinite(hi).all()):
                b = int(log2_brick)
                lo_i = [(int(v) >> b) << b for v in lo.tolist()]
                span = max(int(h) - l for h, l in zip(hi.tolist(), lo_i)) + 1
                bits = max(b, (span - 1).bit_length())
                if bits <= 10:
                    k32 = torch.empty(n, dtype=torch.int32, device=pts.device)
                    _native.check(lib.sp_morton_keys32(pts.data_ptr(), n, dtype, lo_i[0], lo_i[1], lo_i[2], bits,
                                                       k32.data_ptr(), st.cuda_stream))
                    keys, perm = torch.sort(k32)
        if keys is None:
            keys = torch.empty(n, dtype=torch.int64, device=pts.device)
            _native.check(lib.sp_morton_keys(pts.data_ptr(), n, dtype, keys.data_ptr(), st.cuda_stream))
            if not presorted:
                keys, perm = torch.sort(keys)
        if perm is not None:
            sp = torch.empty_like(pts)
            _native.check(lib.sp_gather_points(pts.data_ptr(), perm.data_ptr(), n, dtype, sp.data_ptr(), st.cuda_stream))
            pts = sp
        # brick runs (points not actually in Morton order just give many short runs:
        # still correct, only slower)
        bid = keys >> (3 * int(log2_brick))
        _, counts = torch.unique_consecutive(bid, return_counts=True)
        start = torch.zeros(counts.shape[0] + 1, dtype=torch.int64, device=pts.device)
        torch.cumsum(counts, 0, out=start[1:])
    return PointBatch(pts, start, log2_brick, perm)


def morton_order(pts: torch.Tensor, stream: torch.cuda.Stream | None = None) -> torch.Tensor:
    """Permutation sorting points by the Morton code of their unit cell floor(x)."""
    lib = _native.lib()
    st = stream if stream is not None else torch.cuda.current_stream(pts.device)
    n = pts.shape[0]
    keys = torch.empty(n, dtype=torch.int64, device=pts.device)
    dtype = _native.SP_F32 if pts.dtype == torch.float32 else _native.SP_F64
    _native.check(lib.sp_morton_keys(pts.data_ptr(), n, dtype, keys.data_ptr(), st.cuda_stream))
    # keys < 2^63, so the signed sort is the unsigned order
    return torch.sort(keys, stable=True).indices
