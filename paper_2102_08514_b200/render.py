"""Volume ray-marcher — the consumer after reconstruction.

SPEC.md's `render_volume(job: RenderJob) -> image` (the reference describes it but does not
ship it): a front-to-back alpha-composited ORTHOGRAPHIC raycast through a lattice volume,
a piecewise-linear transfer function (colour + opacity over the value range), a fixed step
size, deterministic output, written as a portable pixmap.  The paper's benchmark setting
(§5.1) is the Marschner–Lobb test signal (f_M = 6, alpha = 0.25) sampled at every lattice
site and reconstructed by the spline under test.

Every sample of every ray is reconstructed by the same GPU kernels as the benchmark
(`PlanInterpreter.eval_batch`), one slab of `slab` steps for all pixels at a time: the
slab's points are generated on the GPU (`sp_ray_points`, csrc/sp_render.cu) pixel-major
with the steps of one ray contiguous, so each CTA's chunk of consecutive points covers a
few short parallel ray segments — a compact staged box (the coherent access pattern of ray
marching the paper's kernels target) — and composited front to back on the
GPU (`sp_composite`, float64 per-pixel state).  `ray_points` is the host definition of the
sample points (the device kernel reproduces it bit for bit); the tests composite the
oracle's reconstruction of the same points with oracle/render_numpy.py and compare.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field
from typing import Sequence

import numpy as np
import torch

from . import _native
from .convergence import sample_grid, spline_center
from .runtime import CoefficientGrid, PlanInterpreter


def marschner_lobb(f_m: float = 6.0, alpha: float = 0.25):
    """The Marschner–Lobb signal on [-1, 1]^3 (SPEC.md design decision: standard formula,
    f_M = 6, alpha = 0.25): (1 - sin(pi z / 2) + alpha (1 + rho_r(sqrt(x^2 + y^2)))) /
    (2 (1 + alpha)) with rho_r(r) = cos(2 pi f_M cos(pi r / 2))."""

    def f(x: torch.Tensor) -> torch.Tensor:
        r = torch.sqrt(x[:, 0] * x[:, 0] + x[:, 1] * x[:, 1])
        rho = torch.cos(2.0 * math.pi * f_m * torch.cos(math.pi * r / 2.0))
        return (1.0 - torch.sin(math.pi * x[:, 2] / 2.0) + alpha * (1.0 + rho)) / (2.0 * (1.0 + alpha))

    return f


@dataclass
class Camera:
    """Orthographic camera: rays start on the image plane through `position`, spanned by
    the `right` / `up` rows of `orientation`, and travel along its `forward` row; `fov` is
    the world-space width of the view (the height follows the image aspect)."""

    position: tuple = (0.0, 0.0, -1.5)
    orientation: tuple = ((1.0, 0.0, 0.0), (0.0, 1.0, 0.0), (0.0, 0.0, 1.0))  # right, up, forward
    fov: float = 2.2


@dataclass
class TransferFunction:
    """Piecewise-linear (value, r, g, b, alpha) control points, clamped outside."""

    points: tuple = ((0.0, 0.0, 0.0, 0.0, 0.0), (0.45, 0.1, 0.2, 0.9, 0.0), (0.5, 1.0, 0.9, 0.6, 0.35),
                     (0.55, 0.1, 0.2, 0.9, 0.0), (1.0, 0.0, 0.0, 0.0, 0.0))

    def __post_init__(self):
        vals = [p[0] for p in self.points]
        if len(self.points) < 2 or any(b <= a for a, b in zip(vals, vals[1:])):
            raise ValueError("transfer function needs >= 2 control points with increasing values")


@dataclass
class RenderJob:
    """SPEC.md RenderJob: plan, volume, camera, image extents, transfer function, step size.
    World point x maps to lattice coordinates x * lattice_scale + lattice_offset (the volume
    helpers below fill sites m with f(m / lattice_scale))."""

    plan: object
    volume: CoefficientGrid
    camera: Camera = field(default_factory=Camera)
    width: int = 256
    height: int = 256
    transfer: TransferFunction = field(default_factory=TransferFunction)
    step: float = 0.01
    n_steps: int = 300
    lattice_scale: float = 1.0
    lattice_offset: tuple = (0.0, 0.0, 0.0)
    background: tuple = (0.0, 0.0, 0.0)
    slab: int = 64

    def __post_init__(self):
        if not self.step > 0:
            raise ValueError("step size must be positive")
        if self.width <= 0 or self.height <= 0 or self.n_steps <= 0:
            raise ValueError("image extents and step count must be positive")


@dataclass
class RenderResult:
    image: np.ndarray          # (height, width, 3) uint8
    radiance: torch.Tensor     # (height, width, 3) float, before quantisation
    samples: int               # reconstructions performed
    ms: float                  # GPU time of the whole render (CUDA events)


def ml_volume(plan, resolution: int, *, device=None, dtype=torch.float32, f_m: float = 6.0, alpha: float = 0.25,
              boundary: str = "zero") -> tuple:
    """Marschner–Lobb sampled on the plan's lattice at spacing h = 2 / resolution over
    [-1, 1]^3 (+ the spline's support).  Returns (grid, lattice_scale, lattice_offset)."""
    from .lattice import decompose_cartesian, named_lattice

    device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    cos = decompose_cartesian(named_lattice(plan.lattice_name))
    h = 2.0 / resolution
    grid = sample_grid(cos, marschner_lobb(f_m, alpha), h, 1.0, 4 + max(cos.diag), device=device, dtype=dtype,
                       boundary=boundary)
    return grid, 1.0 / h, spline_center(plan)


def ray_points(job: RenderJob, k0: int, k1: int, device, dtype) -> torch.Tensor:
    """Lattice-coordinate sample points of steps [k0, k1) of every ray, pixel-major with the
    steps of one ray contiguous: ((height * width * (k1 - k0)), 3)."""
    cam = job.camera
    R = torch.tensor(cam.orientation, dtype=torch.float64, device=device)
    right, up, fwd = R[0], R[1], R[2]
    w, h = job.width, job.height
    u = (torch.arange(w, dtype=torch.float64, device=device) + 0.5) / w - 0.5
    v = 0.5 - (torch.arange(h, dtype=torch.float64, device=device) + 0.5) / h
    span_y = cam.fov * h / w
    org = (torch.tensor(cam.position, dtype=torch.float64, device=device)
           + (v[:, None, None] * span_y) * up + (u[None, :, None] * cam.fov) * right)  # (h, w, 3)
    t = (torch.arange(k0, k1, dtype=torch.float64, device=device) + 0.5) * job.step
    p = org[:, :, None, :] + t[None, None, :, None] * fwd  # (h, w, s, 3) world
    off = torch.tensor(job.lattice_offset, dtype=torch.float64, device=device)
    return (p * job.lattice_scale + off).reshape(-1, 3).to(dtype)


def finish(state, background: Sequence[float], height: int, width: int) -> tuple:
    col, trans = state
    bg = torch.tensor(background, dtype=torch.float64, device=col.device)
    rad = (col + trans[:, None] * bg).reshape(height, width, 3)
    img = (rad.clamp(0.0, 1.0) * 255.0 + 0.5).floor().to(torch.uint8)
    return rad, img.cpu().numpy()


def _camera_desc(job: RenderJob) -> _native.Camera:
    cam = _native.Camera()
    R = job.camera.orientation
    for a in range(3):
        cam.position[a] = float(job.camera.position[a])
        cam.right[a] = float(R[0][a])
        cam.up[a] = float(R[1][a])
        cam.forward[a] = float(R[2][a])
        cam.lattice_offset[a] = float(job.lattice_offset[a])
    cam.fov = float(job.camera.fov)
    cam.step = float(job.step)
    cam.lattice_scale = float(job.lattice_scale)
    return cam


def _transfer_desc(tf: TransferFunction) -> _native.Transfer:
    if len(tf.points) > _native.SP_MAX_TRANSFER:
        raise ValueError(f"at most {_native.SP_MAX_TRANSFER} transfer-function control points")
    d = _native.Transfer()
    d.n = len(tf.points)
    for i, pt in enumerate(tf.points):
        for j in range(5):
            d.points[5 * i + j] = float(pt[j])
    return d


def render_volume(job: RenderJob, interp: PlanInterpreter | None = None) -> RenderResult:
    """SPEC.md render_volume: per slab of steps, the rays' sample points (sp_ray_points),
    their reconstruction (eval_batch, chunk kernel) and front-to-back compositing
    (sp_composite), all on the GPU and stream-ordered; one host sync at the end."""
    interp = interp or PlanInterpreter(job.plan)
    grid = job.volume
    dev = grid.device
    if dev.type != "cuda":
        raise RuntimeError("render_volume needs the volume on a CUDA device")
    lib = _native.lib()
    cam, tfd = _camera_desc(job), _transfer_desc(job.transfer)
    npx = job.width * job.height
    slab = min(job.slab, job.n_steps)
    pts = torch.empty((npx * slab, 3), dtype=torch.float32, device=dev)
    vals = torch.empty(npx * slab, dtype=grid.dtype, device=dev)
    state = torch.zeros((npx, 4), dtype=torch.float64, device=dev)
    state[:, 3] = 1.0
    dt = _native.SP_F32 if grid.dtype == torch.float32 else _native.SP_F64
    stream = torch.cuda.current_stream(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for k0 in range(0, job.n_steps, slab):
        k1 = min(job.n_steps, k0 + slab)
        m = npx * (k1 - k0)
        _native.check(lib.sp_ray_points(ctypes.byref(cam), job.width, job.height, k0, k1, pts.data_ptr(),
                                        ctypes.c_void_p(stream.cuda_stream)))
        p = pts[:m] if grid.dtype == torch.float32 else pts[:m].to(grid.dtype)
        interp.eval_batch(grid, p, out=vals[:m], check=False, order="given", stream=stream)  # coherent by construction
        _native.check(lib.sp_composite(vals.data_ptr(), dt, npx, k1 - k0, ctypes.byref(tfd), state.data_ptr(),
                                       ctypes.c_void_p(stream.cuda_stream)))
    rad, img = finish((state[:, :3], state[:, 3]), job.background, job.height, job.width)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    return RenderResult(image=img, radiance=rad, samples=npx * job.n_steps, ms=e0.elapsed_time(e1))


def write_ppm(path: str, image: np.ndarray) -> None:
    """Binary portable pixmap (P6), as the SPEC's render verb writes."""
    h, w, _ = image.shape
    with open(path, "wb") as fh:
        fh.write(f"P6\n{w} {h}\n255\n".encode())
        fh.write(np.ascontiguousarray(image, dtype=np.uint8).tobytes())


def read_ppm(path: str) -> np.ndarray:
    with open(path, "rb") as fh:
        data = fh.read()
    parts = data.split(b"\n", 3)
    if parts[0] != b"P6":
        raise ValueError("not a binary PPM")
    w, h = (int(v) for v in parts[1].split())
    return np.frombuffer(parts[3], dtype=np.uint8).reshape(h, w, 3)


def main(argv=None) -> None:
    """python -m paper_2102_08514_b200.render --plan cc_tricubic --res 64 --out ml.ppm"""
    import argparse

    from . import corpus

    ap = argparse.ArgumentParser(description=main.__doc__)
    ap.add_argument("--plan", default="cc_tricubic")
    ap.add_argument("--res", type=int, default=64, help="lattice samples across [-1, 1]")
    ap.add_argument("--size", type=int, default=512)
    ap.add_argument("--steps", type=int, default=384)
    ap.add_argument("--out", default="ml.ppm")
    a = ap.parse_args(argv)
    plan = corpus.build_plan(a.plan)
    grid, sc, off = ml_volume(plan, a.res)
    job = RenderJob(plan=plan, volume=grid, width=a.size, height=a.size, n_steps=a.steps, step=3.0 / a.steps,
                    lattice_scale=sc, lattice_offset=off)
    res = render_volume(job)
    write_ppm(a.out, res.image)
    print(f"{a.plan} res={a.res}: {res.samples} samples in {res.ms:.2f} ms "
          f"({res.samples / res.ms / 1e6:.2f} Gsamples/s) -> {a.out}")


if __name__ == "__main__":
    main()
