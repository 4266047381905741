"""Ray-marcher (render.py, SPEC.md render_volume): host logic on CPU, renders on the GPU.

GPU renders are checked against the same compositing applied to the numpy oracle's
reconstruction of every ray sample (oracle/plan_numpy.py, pinned to the reference), plus
the SPEC's examples: an all-zero volume renders the background; a constant volume with an
opaque transfer at that value renders the silhouette of the domain box."""
import numpy as np
import pytest
import torch

from paper_2102_08514_b200 import corpus
from oracle.render_numpy import composite, finish, transfer
from paper_2102_08514_b200.render import (Camera, RenderJob, TransferFunction, marschner_lobb, ml_volume, ray_points,
                                          read_ppm, render_volume, write_ppm)


def test_transfer_function_is_piecewise_linear_and_clamped():
    tf = TransferFunction(((0.0, 0, 0, 0, 0.0), (1.0, 1, 0.5, 0, 1.0)))
    rgb, a = transfer(tf.points, np.array([-1.0, 0.0, 0.25, 1.0, 3.0]))
    assert a.tolist() == [0.0, 0.0, 0.25, 1.0, 1.0]
    assert rgb[2].tolist() == [0.25, 0.125, 0.0]
    with pytest.raises(ValueError):
        TransferFunction(((0.0, 0, 0, 0, 0), (0.0, 1, 1, 1, 1)))


def test_composite_slabs_compose():
    rng = np.random.default_rng(1)
    vals = rng.random((7, 23))
    tf = TransferFunction()
    s = composite(vals[:, 10:], tf.points, composite(vals[:, :10], tf.points))
    whole = composite(vals, tf.points)
    np.testing.assert_allclose(s[0], whole[0], rtol=1e-13, atol=1e-15)
    np.testing.assert_allclose(s[1], whole[1], rtol=1e-13, atol=1e-15)


def test_ray_points_geometry():
    plan = corpus.build_plan("cc_trilinear")
    job = RenderJob(plan=plan, volume=None, width=4, height=2, step=0.5, n_steps=3, lattice_scale=2.0,
                    lattice_offset=(1.0, 1.0, 1.0), camera=Camera(position=(0, 0, -1), fov=2.0))
    p = ray_points(job, 0, 3, "cpu", torch.float64).reshape(2, 4, 3, 3)
    # pixel (0, 0): u = -0.375 * 2, v = +0.25 * 1 (height spans fov * 2 / 4 = 1); steps at t = 0.25, 0.75, 1.25
    want0 = np.array([[-0.75, 0.25, -1 + t] for t in (0.25, 0.75, 1.25)]) * 2.0 + 1.0
    np.testing.assert_allclose(p[0, 0].numpy(), want0)
    assert torch.all(p[1, :, :, 1] < p[0, :, :, 1])  # image rows go down


def test_ppm_roundtrip(tmp_path):
    img = np.random.default_rng(2).integers(0, 256, (5, 7, 3), dtype=np.uint8)
    write_ppm(str(tmp_path / "a.ppm"), img)
    np.testing.assert_array_equal(read_ppm(str(tmp_path / "a.ppm")), img)


def test_marschner_lobb_range():
    x = torch.from_numpy(np.random.default_rng(3).uniform(-1, 1, (1000, 3)))
    v = marschner_lobb()(x)
    assert float(v.min()) >= 0.0 and float(v.max()) <= 1.0


@pytest.mark.gpu
def test_zero_volume_renders_background(cuda):
    plan = corpus.build_plan("bcc_linear_rd")
    grid, sc, off = ml_volume(plan, 16, device=cuda)
    for a in grid.arrays:
        a.zero_()
    job = RenderJob(plan=plan, volume=grid, width=16, height=12, n_steps=64, step=0.05, lattice_scale=sc,
                    lattice_offset=off, background=(0.2, 0.4, 0.6))
    res = render_volume(job)
    assert (res.image == np.array([51, 102, 153], np.uint8)).all()


@pytest.mark.gpu
def test_constant_volume_renders_box_silhouette(cuda):
    plan = corpus.build_plan("cc_tricubic")
    grid, sc, off = ml_volume(plan, 16, device=cuda)
    # constant 1 on the sites covering [-1, 1]^3 (+ margin): partition of unity inside
    for a in grid.arrays:
        a.fill_(1.0)
    tf = TransferFunction(((0.0, 1, 1, 1, 0.0), (0.9, 1, 1, 1, 0.0), (1.0, 1, 1, 1, 1.0)))  # white, opaque at 1
    job = RenderJob(plan=plan, volume=grid, width=40, height=40, n_steps=160, step=0.025, lattice_scale=sc,
                    lattice_offset=off, transfer=tf, camera=Camera(position=(0, 0, -2), fov=4.0))
    img = render_volume(job).image
    assert (img[20, 20] == 255).all() and (img[0, 0] == 0).all() and (img[39, 39] == 0).all()
    lit = (img[:, :, 0] == 255)
    rows = np.flatnonzero(lit.any(1))
    cols = np.flatnonzero(lit.any(0))
    # the box is symmetric about the view axis and its lit region is a solid rectangle
    assert rows[0] + rows[-1] == 39 and cols[0] + cols[-1] == 39
    assert lit[rows[0]:rows[-1] + 1, cols[0]:cols[-1] + 1].all()


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["cc_trilinear", "bcc_linear_rd", "fcc_cubic"])
def test_render_matches_oracle_composite(name, cuda):
    from oracle.plan_numpy import NumpyGrid, PlanTables, eval_batch as oracle_eval

    plan = corpus.build_plan(name)
    grid, sc, off = ml_volume(plan, 12, device=cuda)
    job = RenderJob(plan=plan, volume=grid, width=20, height=16, n_steps=48, step=0.06, lattice_scale=sc,
                    lattice_offset=off, slab=20, camera=Camera(position=(0.1, -0.05, -1.4), fov=2.4))
    res = render_volume(job)
    ngrid = NumpyGrid(plan.diag, plan.shifts, [a.double().cpu().numpy() for a in grid.arrays], grid.origins)
    tables = PlanTables(plan)
    state = None
    npx = job.width * job.height
    for k0 in range(0, job.n_steps, job.slab):
        k1 = min(job.n_steps, k0 + job.slab)
        pts = ray_points(job, k0, k1, "cpu", torch.float32).double().numpy()
        vals = oracle_eval(plan, ngrid, pts, tables).reshape(npx, k1 - k0)
        state = composite(vals, job.transfer.points, state)
    rad, img = finish(state, job.background, job.height, job.width)
    assert float(rad.max()) > 0.05  # the transfer function picks up the ML structure
    np.testing.assert_allclose(res.radiance.cpu().numpy(), rad, rtol=0, atol=2e-4)
    assert int(np.abs(res.image.astype(int) - img.astype(int)).max()) <= 1


@pytest.mark.gpu
def test_device_ray_points_equal_host_definition(cuda):
    import ctypes

    from paper_2102_08514_b200 import _native
    from paper_2102_08514_b200.render import _camera_desc

    plan = corpus.build_plan("bcc_linear_rd")
    job = RenderJob(plan=plan, volume=None, width=37, height=23, n_steps=50, step=0.037, lattice_scale=13.7,
                    lattice_offset=(1.0, 1.0, 1.0),
                    camera=Camera(position=(0.3, -0.2, -1.7), fov=2.3,
                                  orientation=((0.8, 0.6, 0.0), (-0.36, 0.48, 0.8), (0.48, -0.64, 0.6))))
    want = ray_points(job, 11, 50, "cpu", torch.float32)
    got = torch.empty_like(want, device=cuda)
    _native.check(_native.lib().sp_ray_points(ctypes.byref(_camera_desc(job)), job.width, job.height, 11, 50,
                                              got.data_ptr(), None))
    torch.cuda.synchronize()
    assert torch.equal(got.cpu(), want)
