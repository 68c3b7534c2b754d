"""The drop-in boundary driven by the reference's own objects.

The reference package (convexsplat 0.1.0) is imported from its offline
install (baseline/_ref, `pip install --target`) or its source tree; the tests
skip when neither exists.  Scenes, cameras, settings and scaling modes are
the reference's own classes (convexsplat.model / rasterize / field); the
reference's rasterize.render / backward.backward are patched with this
package's drop-in, as INTEGRATION.md's option 1 does, and the reference's
known-answer cases (tests/test_rasterize.py, tests/test_backward.py of the
reference, restated here with their line numbers) run through it on the
GPU.  Tolerances are the float32 contract (1e-4 images) where
the reference asserts float64 identities.
"""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for _p in (os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"):
    if os.path.isdir(os.path.join(_p, "convexsplat")) and _p not in sys.path:
        sys.path.append(_p)
        break
ref = pytest.importorskip("convexsplat")
import importlib  # noqa: E402

# the modules (the package re-exports functions of the same names)
ref_backward = importlib.import_module("convexsplat.backward")
ref_rasterize = importlib.import_module("convexsplat.rasterize")
from convexsplat.field import ScalingMode as RefMode  # noqa: E402
from convexsplat.harmonics import SH_C0  # noqa: E402
from convexsplat.model import (Camera, Scene, SmoothConvex, inverse_delta_activation,  # noqa: E402
                               inverse_mask_activation, inverse_opacity_activation, inverse_sigma_activation)
from convexsplat.synth import make_scene, ring_cameras  # noqa: E402

ATOL = 1e-4


def ortho_camera(size=48):
    """test_rasterize.py:21-23"""
    return Camera(fx=1.0, fy=1.0, cx=0.0, cy=0.0, width=size, height=size, R=np.eye(3), t=np.zeros(3), ortho=True)


def hexagon(center_xy, z, opacity, color, radius=20.0, sigma=2.5):
    """test_rasterize.py:33-46: a flat hexagon whose interior indicator saturates."""
    ang = np.linspace(0.0, 2 * np.pi, 7)[:-1]
    pts = np.stack([center_xy[0] + radius * np.cos(ang), center_xy[1] + radius * np.sin(ang), np.full(6, float(z))],
                   axis=1)
    sh = np.zeros((16, 3))
    sh[0] = (np.asarray(color, dtype=float) - 0.5) / SH_C0
    return SmoothConvex(points=pts, raw_delta=inverse_delta_activation(1.0), raw_sigma=inverse_sigma_activation(sigma),
                        raw_opacity=inverse_opacity_activation(opacity), sh=sh, raw_mask=inverse_mask_activation(0.999))


def quantize32(scene):
    """The reference scene rounded to the float32 values the GPU stores
    (the quantize32 pattern of the reference's test_sceneio.py:19-29), so
    both sides see identical parameters."""
    for c in scene.primitives:
        c.points = c.points.astype(np.float32).astype(np.float64)
        c.sh = c.sh.astype(np.float32).astype(np.float64)
        for f in ("raw_delta", "raw_sigma", "raw_opacity", "raw_mask"):
            setattr(c, f, float(np.float32(getattr(c, f))))
    return scene


def test_reference_objects_convert_without_a_gpu():
    """CPU: the reference's Scene / Camera / RenderSettings / ScalingMode pass
    the drop-in's conversion (duck typing; no isinstance on this package's
    types) -- scene_tensors.as_scene_tensors, rasterizer.*_struct."""
    from paper_2411_14974_b200 import rasterizer as rz
    from paper_2411_14974_b200.scene_tensors import as_scene_tensors
    scene = make_scene(num_primitives=5, seed=0)
    st = as_scene_tensors(scene, "cpu")
    assert st.n == 5 and st.k == 6
    np.testing.assert_array_equal(st.points.numpy(), np.stack([c.points for c in scene.primitives]).astype(np.float32))
    cam = ring_cameras(2, size=64)[1]
    c = rz.camera_struct(cam)
    assert (c.width, c.height) == (64, 64) and c.fx == cam.fx
    s = rz.settings_struct(ref_rasterize.RenderSettings(), RefMode.SQRT_DEPTH, scene.background)
    assert s.scaling_mode == 1 and s.cutoff == 2e-4 and s.tile == 16


@pytest.fixture
def dropin(monkeypatch):
    """The reference's render / render_reference / backward replaced by the
    drop-in (INTEGRATION.md option 1)."""
    import paper_2411_14974_b200 as cs
    monkeypatch.setattr(ref_rasterize, "render", cs.render)
    monkeypatch.setattr(ref_rasterize, "render_reference", cs.render_reference)
    monkeypatch.setattr(ref_backward, "backward", cs.backward)
    return cs


@pytest.mark.gpu
def test_empty_scene_renders_background(dropin):
    """test_rasterize.py:48-55"""
    bg = np.array([0.2, 0.4, 0.6])
    out = ref_rasterize.render(Scene([], background=bg), ortho_camera(), RefMode.NONE)
    np.testing.assert_allclose(out.image, np.broadcast_to(bg, out.image.shape), atol=1e-7)
    assert np.all(out.final_transmittance == 1.0) and np.all(out.per_pixel_count == 0)
    assert np.all(out.blend_weight_sum == 0.0)


@pytest.mark.gpu
def test_saturated_single_primitive_center_pixel(dropin):
    """test_rasterize.py:58-69: interior alpha is the opacity."""
    color = (1.0, 0.5, 0.0)
    out = ref_rasterize.render(Scene([hexagon((24.5, 24.5), 2.0, 0.5, color)], background=np.zeros(3)),
                               ortho_camera(), RefMode.NONE)
    assert abs(out.blend_weight_sum[24, 24] - 0.5) < 1e-6
    assert abs(out.final_transmittance[24, 24] - 0.5) < 1e-6
    assert out.per_pixel_count[24, 24] == 1
    np.testing.assert_allclose(out.image[24, 24], 0.5 * np.array(color), atol=1e-6)


@pytest.mark.gpu
def test_two_primitive_front_to_back_weights(dropin):
    """test_rasterize.py:72-83: 0.5 c_front + 0.25 c_back + 0.25 bg."""
    bg = np.array([0.1, 0.1, 0.1])
    cf, cb = (1.0, 0.0, 0.0), (0.0, 1.0, 0.0)
    scene = Scene([hexagon((24.5, 24.5), 3.0, 0.5, cb), hexagon((24.5, 24.5), 2.0, 0.5, cf)], background=bg)
    out = ref_rasterize.render(scene, ortho_camera(), RefMode.NONE)
    assert abs(out.blend_weight_sum[24, 24] - 0.75) < 1e-6
    assert abs(out.final_transmittance[24, 24] - 0.25) < 1e-6
    np.testing.assert_allclose(out.image[24, 24], 0.5 * np.array(cf) + 0.25 * np.array(cb) + 0.25 * bg, atol=1e-6)


@pytest.mark.gpu
def test_depth_order_and_equal_depth_tie(dropin):
    """test_rasterize.py:86-105: blending follows depth, not list order; an
    equal-depth tie is broken by scene index."""
    cam = ortho_camera()
    front = hexagon((24.5, 24.5), 2.0, 0.5, (1.0, 0.0, 0.0))
    back = hexagon((24.5, 24.5), 3.0, 0.5, (0.0, 1.0, 0.0))
    a = ref_rasterize.render(Scene([front, back], background=np.zeros(3)), cam, RefMode.NONE)
    b = ref_rasterize.render(Scene([back, front], background=np.zeros(3)), cam, RefMode.NONE)
    np.testing.assert_array_equal(a.image, b.image)
    assert a.image[24, 24, 0] > a.image[24, 24, 1]
    red = hexagon((24.5, 24.5), 2.0, 0.5, (1.0, 0.0, 0.0))
    green = hexagon((24.5, 24.5), 2.0, 0.5, (0.0, 1.0, 0.0))
    out = ref_rasterize.render(Scene([red, green], background=np.zeros(3)), cam, RefMode.NONE)
    assert abs(out.image[24, 24, 0] - 0.5) < 1e-6 and abs(out.image[24, 24, 1] - 0.25) < 1e-6


@pytest.mark.gpu
def test_compositing_identity(dropin):
    """test_rasterize.py:108-116: blend_weight_sum + final T == 1."""
    for seed in range(3):
        scene = make_scene(num_primitives=6, seed=seed)
        cam = ring_cameras(4, size=64)[seed % 4]
        for settings in (ref_rasterize.EXACT_SETTINGS, ref_rasterize.RenderSettings()):
            out = ref_rasterize.render(scene, cam, RefMode.DEPTH, settings)
            np.testing.assert_allclose(out.blend_weight_sum + out.final_transmittance, 1.0, atol=1e-6)


@pytest.mark.gpu
def test_exact_and_production_against_the_reference_itself(dropin, monkeypatch):
    """test_rasterize.py:118-139: the drop-in's EXACT render against the
    reference's own render_reference (float64 NumPy) within the float32 bar
    (the reference pins its two float64 paths bit-equal), and the production
    settings within the reference's 2/255 quantisation bound."""
    monkeypatch.undo()        # the unpatched reference for the ground truth
    import paper_2411_14974_b200 as cs
    worst = 0.0
    for seed in range(3):
        scene = make_scene(num_primitives=7, seed=10 + seed)
        cam = ring_cameras(4, size=64)[seed % 4]
        want = ref_rasterize.render_reference(scene, cam, RefMode.DEPTH)
        got = cs.render(scene, cam, RefMode.DEPTH, ref_rasterize.EXACT_SETTINGS)
        for f in ("image", "final_transmittance", "blend_weight_sum"):
            np.testing.assert_allclose(getattr(got, f), getattr(want, f), rtol=0, atol=ATOL)
        np.testing.assert_array_equal(got.per_pixel_count, want.per_pixel_count)
        prod = cs.render(scene, cam, RefMode.DEPTH)
        worst = max(worst, float(np.abs(prod.image - want.image).max()))
    assert worst <= 2.0 / 255.0


@pytest.mark.gpu
def test_alpha_cap_keeps_transmittance_positive(dropin):
    """test_rasterize.py:188-194"""
    conv = hexagon((24.5, 24.5), 2.0, 0.5, (1.0, 1.0, 1.0))
    conv.raw_opacity = 40.0
    out = ref_rasterize.render(Scene([conv], background=np.zeros(3)), ortho_camera(), RefMode.NONE)
    assert np.all(out.final_transmittance > 0.0)
    assert abs(out.final_transmittance[24, 24] - (1.0 - ref_rasterize.ALPHA_MAX)) < 1e-9


@pytest.mark.gpu
def test_backward_known_answers(dropin):
    """test_backward.py:69-126 through the patched reference backward: zero
    in -> zero out, GradientBuffer.add linearity, red-channel isolation, an
    interior point gets no gradient, visibility equals the renderer's."""
    scene = make_scene(num_primitives=2, seed=3)
    cam = ring_cameras(4, size=32)[0]
    g = ref_backward.backward(scene, cam, np.zeros((32, 32, 3)), RefMode.DEPTH)
    assert np.all(ref_backward.pack_grads(g) == 0.0) and g.visible.any()
    scene = make_scene(num_primitives=2, seed=4)
    d = np.full((32, 32, 3), 0.5)
    once = ref_backward.backward(scene, cam, d, RefMode.DEPTH)
    twice = ref_backward.backward(scene, cam, d, RefMode.DEPTH)
    twice.add(ref_backward.backward(scene, cam, d, RefMode.DEPTH))
    a, b = ref_backward.pack_grads(twice), 2 * ref_backward.pack_grads(once)
    assert np.abs(a - b).max() <= 1e-6 * np.abs(b).max()     # float atomics: summation order
    ocam = ortho_camera()
    conv = hexagon((24.5, 24.5), 2.0, 0.6, (0.8, 0.3, 0.1))
    d_image = np.zeros((48, 48, 3))
    d_image[..., 0] = 1.0
    g = ref_backward.backward(Scene([conv], background=np.zeros(3)), ocam, d_image, RefMode.NONE)
    assert g.d_sh[0, 0, 0] > 0.0 and np.all(g.d_sh[0, :, 1:] == 0.0) and g.d_raw_opacity[0] > 0.0
    conv2 = conv.copy()
    conv2.points = np.vstack([conv.points, [[24.5, 24.5, 2.0]]])
    d_image = np.random.default_rng(0).normal(size=(48, 48, 3))
    g = ref_backward.backward(Scene([conv2], background=np.zeros(3)), ocam, d_image, RefMode.NONE,
                              ref_rasterize.RenderSettings(sh_degree=0))
    np.testing.assert_array_equal(g.d_points[0, 6], 0.0)
    assert np.abs(g.d_points[0, :6, :2]).max() > 0.0
    scene = make_scene(num_primitives=6, seed=5)
    g = ref_backward.backward(scene, cam, np.ones((32, 32, 3)), RefMode.DEPTH)
    np.testing.assert_array_equal(g.visible, ref_rasterize.render(scene, cam, RefMode.DEPTH).visible)


@pytest.mark.gpu
def test_prepare_view_and_bin_tiles_drop_in(dropin):
    """prepare_view (rasterize.py:77-122) returns the reference's full
    ProjectedConvex / ViewPrimitive fields, equal to the reference's own
    (discrete state exactly, float64 geometry to 1e-9), and bin_tiles
    (rasterize.py:134-144) accepts both this package's and the reference's
    prepared lists; the reference CLI overlay (cli.py:290-305) reads
    vp.pc.pixels[vp.pc.hull_indices]."""
    import paper_2411_14974_b200 as cs
    scene = quantize32(make_scene(num_primitives=12, seed=7))
    cam = ring_cameras(4, size=96)[2]
    want = ref_rasterize.prepare_view(scene, cam, RefMode.DEPTH, ref_rasterize.RenderSettings())
    got = cs.prepare_view(scene, cam, RefMode.DEPTH, ref_rasterize.RenderSettings())
    assert [vp.pc.index for vp in got] == [vp.pc.index for vp in want]
    for g, w in zip(got, want):
        np.testing.assert_array_equal(g.pc.hull_indices, w.pc.hull_indices)
        assert tuple(g.pc.bbox) == tuple(w.pc.bbox) and g.pc.depth == w.pc.depth
        np.testing.assert_array_equal(g.pc.pixels, w.pc.pixels)
        np.testing.assert_array_equal(g.pc.point_depths, w.pc.point_depths)
        np.testing.assert_array_equal(g.pc.normals, w.pc.normals)
        np.testing.assert_array_equal(g.pc.offsets, w.pc.offsets)
        np.testing.assert_allclose([g.pc.delta_s, g.pc.sigma_s, g.opacity, g.scale, g.view_dist],
                                   [w.pc.delta_s, w.pc.sigma_s, w.opacity, w.scale, w.view_dist], rtol=1e-12)
        np.testing.assert_allclose(g.view_dir, w.view_dir, rtol=0, atol=1e-14)
        np.testing.assert_allclose(g.color, w.color, rtol=0, atol=1e-12)
        assert g.pc.hull_pixels.shape == w.pc.hull_pixels.shape
    want_bins = ref_rasterize.bin_tiles(want, 96, 96, 16)
    assert cs.bin_tiles(got, 96, 96, 16) == want_bins
    assert cs.bin_tiles(want, 96, 96, 16) == want_bins        # the reference's own prepared list
