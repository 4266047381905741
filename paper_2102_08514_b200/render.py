"""Volume ray-marcher — the consumer after reconstruction.

SPEC.md's `render_volume(job: RenderJob) -> image` (the reference describes it but does not
ship it): a front-to-back alpha-composited ORTHOGRAPHIC raycast through a lattice volume,
a piecewise-linear transfer function (colour + opacity over the value range), a fixed step
size, deterministic output, written as a portable pixmap.  The paper's benchmark setting
(§5.1) is the Marschner–Lobb test signal (f_M = 6, alpha = 0.25) sampled at every lattice
site and reconstructed by the spline under test.

Every sample of every ray is reconstructed by the same GPU kernels as the benchmark
(`PlanInterpreter.eval_batch`), one slab of `slab` steps for all pixels at a time: the
slab's points are laid out pixel-major with the steps of one ray contiguous, so each CTA's
chunk of consecutive points covers a few short parallel ray segments — a compact staged
box (the coherent access pattern of ray marching the paper's kernels target).
Compositing is a per-slab exclusive cumulative product of transmittance on the GPU; the
same `composite` code runs on CPU tensors, which is how the tests check a GPU render
against one composited from the oracle's values.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Sequence

import numpy as np
import torch

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

    def apply(self, v: torch.Tensor) -> tuple:
        """(rgb (..., 3), alpha (...)) for values v."""
        tab = torch.tensor(self.points, dtype=v.dtype, device=v.device)
        xs = tab[:, 0].contiguous()
        vc = v.clamp(float(xs[0]), float(xs[-1]))
        i = torch.searchsorted(xs, vc.contiguous(), right=True).clamp(1, len(self.points) - 1)
        x0, x1 = xs[i - 1], xs[i]
        w = ((vc - x0) / (x1 - x0)).unsqueeze(-1)
        out = tab[i - 1, 1:] + w * (tab[i, 1:] - tab[i - 1, 1:])
        return out[..., :3], out[..., 3]


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


def composite(values: torch.Tensor, transfer: TransferFunction, state=None):
    """Front-to-back compositing of one slab: values (pixels, steps).  state = (colour
    (pixels, 3), transmittance (pixels,)); returns the updated state.  Deterministic: an
    exclusive cumulative product along each ray, no atomics."""
    rgb, a = transfer.apply(values.to(torch.float64))
    npx = values.shape[0]
    if state is None:
        state = (torch.zeros((npx, 3), dtype=torch.float64, device=values.device),
                 torch.ones(npx, dtype=torch.float64, device=values.device))
    col, trans = state
    keep = 1.0 - a
    excl = torch.cumprod(torch.cat([torch.ones_like(keep[:, :1]), keep[:, :-1]], 1), 1)  # prod_{j<i}
    wgt = trans[:, None] * excl * a
    col = col + (wgt[:, :, None] * rgb).sum(1)
    trans = trans * torch.prod(keep, 1)
    return col, trans


def finish(state, background: Sequence[float], height: int, width: int) -> tuple:
    col, trans = state
    bg = torch.tensor(background, dtype=torch.float64, device=col.device)
    rad = (col + trans[:, None] * bg).reshape(height, width, 3)
    img = (rad.clamp(0.0, 1.0) * 255.0 + 0.5).floor().to(torch.uint8)
    return rad, img.cpu().numpy()


def render_volume(job: RenderJob, interp: PlanInterpreter | None = None) -> RenderResult:
    """SPEC.md render_volume: every ray sample reconstructed on the GPU, composited front to
    back.  Raises RuntimeError_ when the volume does not match the plan's lattice."""
    interp = interp or PlanInterpreter(job.plan)
    grid = job.volume
    dev = grid.device
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    state = None
    npx = job.width * job.height
    for k0 in range(0, job.n_steps, job.slab):
        k1 = min(job.n_steps, k0 + job.slab)
        pts = ray_points(job, k0, k1, dev, grid.dtype)
        vals = interp.eval_batch(grid, pts, check=False).reshape(npx, k1 - k0)
        state = composite(vals, job.transfer, state)
    rad, img = finish(state, job.background, job.height, job.width)
    e1.record()
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
