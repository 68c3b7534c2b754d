"""Generate the golden parity fixtures by running the REFERENCE itself.

Run in the build container only (the reference is not on the GPU box):

    python tests/golden/make_golden.py            # writes tests/golden/*.npz

It imports ``convexsplat`` from /root/reference/pkg/src (read-only) and
records, for a set of seeded scenes/cameras, every hot-path output the
reference exposes: prepare_view (rasterize.py:77-122), bin_tiles
(rasterize.py:134-144), render (rasterize.py:156-209), render_reference
(rasterize.py:212-245) and backward (backward.py:76-212), plus
graham_scan (projection.py:47-113) on the reference test-suite's adversarial
hull generator (tests/oracles.py:67-102).

All scene parameters are first quantised to float32 (the pattern of
tests/test_sceneio.py:19-29) so the float32 GPU path and the float64 oracle
see identical inputs.
"""
from __future__ import annotations

import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
REF_TESTS = "/root/reference/pkg/tests"
sys.path.insert(0, REF_SRC)
sys.path.insert(0, REF_TESTS)
sys.dont_write_bytecode = True

from convexsplat.backward import backward  # noqa: E402
from convexsplat.field import ScalingMode  # noqa: E402
from convexsplat.losses import image_loss  # noqa: E402
from convexsplat.model import (Camera, Scene, SmoothConvex,  # noqa: E402
                               inverse_delta_activation, inverse_mask_activation,
                               inverse_opacity_activation, inverse_sigma_activation)
from convexsplat.projection import graham_scan  # noqa: E402
from convexsplat.rasterize import (EXACT_SETTINGS, RenderSettings, bin_tiles,  # noqa: E402
                                   prepare_view, render, render_reference)
from convexsplat.synth import make_scene, perturb_scene, ring_cameras  # noqa: E402
from oracles import hull_case  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
MODE_NAME = {ScalingMode.NONE: "none", ScalingMode.SQRT_DEPTH: "sqrt",
             ScalingMode.DEPTH: "depth", ScalingMode.DEPTH_SQUARED: "depth2"}


def quantize32(scene: Scene) -> Scene:
    q = scene.copy()
    for c in q.primitives:
        c.points = c.points.astype(np.float32).astype(np.float64)
        c.sh = c.sh.astype(np.float32).astype(np.float64)
        c.raw_delta = float(np.float32(c.raw_delta))
        c.raw_sigma = float(np.float32(c.raw_sigma))
        c.raw_opacity = float(np.float32(c.raw_opacity))
        c.raw_mask = float(np.float32(c.raw_mask))
    return q


def hexagon(center_xy, z, opacity, color, radius=20.0, sigma=2.5, delta=1.0):
    """Same construction as the reference test helper (test_rasterize.py:30-45)."""
    ang = np.linspace(0.0, 2 * np.pi, 7)[:-1]
    pts = np.stack([center_xy[0] + radius * np.cos(ang), center_xy[1] + radius * np.sin(ang),
                    np.full(6, float(z))], axis=1)
    sh = np.zeros((16, 3))
    sh[0] = (np.asarray(color, dtype=float) - 0.5) / 0.28209479177387814
    return SmoothConvex(points=pts, raw_delta=inverse_delta_activation(delta),
                        raw_sigma=inverse_sigma_activation(sigma),
                        raw_opacity=inverse_opacity_activation(opacity), sh=sh,
                        raw_mask=inverse_mask_activation(0.999))


def ortho_camera(size=48):
    return Camera(fx=1.0, fy=1.0, cx=0.0, cy=0.0, width=size, height=size, R=np.eye(3),
                  t=np.zeros(3), ortho=True)


def scene_arrays(scene: Scene) -> dict:
    prims = scene.primitives
    n = len(prims)
    k = prims[0].num_points if n else 6
    return dict(
        points=np.stack([c.points for c in prims]) if n else np.zeros((0, k, 3)),
        raw_delta=np.array([c.raw_delta for c in prims], dtype=np.float64),
        raw_sigma=np.array([c.raw_sigma for c in prims], dtype=np.float64),
        raw_opacity=np.array([c.raw_opacity for c in prims], dtype=np.float64),
        raw_mask=np.array([c.raw_mask for c in prims], dtype=np.float64),
        sh=np.stack([c.sh for c in prims]) if n else np.zeros((0, 16, 3)),
        background=np.asarray(scene.background, dtype=np.float64),
    )


def camera_arrays(cam: Camera) -> dict:
    return dict(cam_intr=np.array([cam.fx, cam.fy, cam.cx, cam.cy, cam.z_near]),
                cam_R=np.asarray(cam.R, dtype=np.float64), cam_t=np.asarray(cam.t, dtype=np.float64),
                cam_size=np.array([cam.width, cam.height, int(cam.ortho)], dtype=np.int64))


def settings_arrays(settings: RenderSettings, mode: ScalingMode) -> dict:
    return dict(set_cut_floor=np.array([settings.contribution_cutoff, settings.transmittance_floor]),
                set_ints=np.array([settings.tile_size, settings.sh_degree], dtype=np.int64),
                set_mode=np.array(MODE_NAME[mode]))


def record(name, scene, cam, mode, settings, d_image=None, reference=False):
    scene = quantize32(scene)
    out = {}
    out.update(scene_arrays(scene))
    out.update(camera_arrays(cam))
    out.update(settings_arrays(settings, mode))
    k = out["points"].shape[1]
    prepared = prepare_view(scene, cam, mode, settings)
    v = len(prepared)
    hull = np.full((v, k), -1, np.int64)
    normals = np.zeros((v, k, 2))
    offsets = np.zeros((v, k))
    for r, vp in enumerate(prepared):
        h = vp.pc.hull_indices.size
        hull[r, :h] = vp.pc.hull_indices
        normals[r, :h] = vp.pc.normals
        offsets[r, :h] = vp.pc.offsets
    out.update(
        prep_index=np.array([vp.pc.index for vp in prepared], dtype=np.int64),
        prep_hull=hull, prep_normals=normals, prep_offsets=offsets,
        prep_bbox=np.array([vp.pc.bbox for vp in prepared], dtype=np.int64).reshape(v, 4),
        prep_depth=np.array([vp.pc.depth for vp in prepared]),
        prep_delta_s=np.array([vp.pc.delta_s for vp in prepared]),
        prep_sigma_s=np.array([vp.pc.sigma_s for vp in prepared]),
        prep_opacity=np.array([vp.opacity for vp in prepared]),
        prep_color=np.array([vp.color for vp in prepared]).reshape(v, 3),
        prep_pixels=np.array([vp.pc.pixels for vp in prepared]).reshape(v, k, 2),
    )
    bins, tx, ty = bin_tiles(prepared, cam.width, cam.height, settings.tile_size)
    out["bin_offsets"] = np.concatenate([[0], np.cumsum([len(b) for b in bins])]).astype(np.int64)
    out["bin_items"] = np.array([i for b in bins for i in b], dtype=np.int64)
    ro = render(scene, cam, mode, settings)
    out.update(img=ro.image, trans=ro.final_transmittance, count=ro.per_pixel_count,
               wsum=ro.blend_weight_sum, visible=ro.visible)
    if reference:
        rr = render_reference(scene, cam, mode)
        out.update(ref_img=rr.image, ref_trans=rr.final_transmittance, ref_count=rr.per_pixel_count,
                   ref_wsum=rr.blend_weight_sum)
    if d_image is not None:
        g = backward(scene, cam, d_image, mode, settings)
        out.update(d_image=d_image, g_points=g.d_points, g_delta=g.d_raw_delta,
                   g_sigma=g.d_raw_sigma, g_opacity=g.d_raw_opacity, g_sh=g.d_sh,
                   g_mask=g.d_raw_mask, g_visible=g.visible)
    path = os.path.join(OUT, f"{name}.npz")
    np.savez_compressed(path, **out)
    print(f"{name}: n={len(scene.primitives)} V={v} P={out['bin_items'].size} -> {path}")


def loss_d_image(scene, cam, mode, settings, seed=1):
    """d_image of the reference training loss against a perturbed target
    (the cli.py:369-378 gradcheck pattern)."""
    scene_q = quantize32(scene)
    target = render(quantize32(perturb_scene(scene, seed=seed)), cam, mode, settings).image
    img = render(scene_q, cam, mode, settings).image
    masks = np.array([c.raw_mask for c in scene_q.primitives])
    return image_loss(img, target, masks).d_image


def gen_hulls():
    pts_all, n_all, hull_all = [], [], []
    cases = [hull_case(i) for i in range(1000)]
    cases += [np.array([[0, 0], [2, 0], [2, 2], [0, 2], [1, 1]], float),
              np.array([[0, 0], [1, 1], [2, 2], [3, 3]], float),
              np.array([[1, 0], [0, 1], [-1, 0], [0, -1], [0.5, -1], [-0.5, -1]], float)]
    maxn = max(c.shape[0] for c in cases)
    for c in cases:
        h = graham_scan(c)
        pad = np.full((maxn, 2), np.nan)
        pad[: c.shape[0]] = c
        pts_all.append(pad)
        n_all.append(c.shape[0])
        hp = np.full(maxn, -1, np.int64)
        if h is not None:
            hp[: h.size] = h
        hull_all.append(hp)
    np.savez_compressed(os.path.join(OUT, "hulls.npz"), points=np.array(pts_all),
                        n=np.array(n_all), hull=np.array(hull_all))
    print(f"hulls: {len(cases)} cases")


def gen_loss():
    """image_loss / ssim_with_grad known answers (losses.py:58-155)."""
    from convexsplat.optim import Adam, position_lr
    rng = np.random.default_rng(7)
    img = rng.uniform(0, 1, size=(23, 31, 3))
    target = np.clip(img + rng.normal(0, 0.1, size=img.shape), 0, 1)
    masks = rng.normal(0, 2, size=17)
    res = image_loss(img, target, masks, 0.2, 0.0005)
    # two Adam steps on a small parameter set (optim.py:12-35)
    params = {"a": rng.normal(size=(5, 3)), "b": rng.normal(size=7)}
    grads1 = {"a": rng.normal(size=(5, 3)), "b": rng.normal(size=7)}
    grads2 = {"a": rng.normal(size=(5, 3)), "b": rng.normal(size=7)}
    p0 = {k: v.copy() for k, v in params.items()}
    adam = Adam({k: v.shape for k, v in params.items()})
    adam.step(params, grads1, {"a": 0.01, "b": 0.002})
    adam.step(params, grads2, {"a": 0.01, "b": 0.002})
    np.savez_compressed(os.path.join(OUT, "loss.npz"), img=img, target=target, masks=masks,
                        total=res.total, l1=res.l1, dssim=res.dssim, mask_term=res.mask_term,
                        d_image=res.d_image, d_raw_mask=res.d_raw_mask,
                        adam_a0=p0["a"], adam_b0=p0["b"], adam_ga1=grads1["a"], adam_gb1=grads1["b"],
                        adam_ga2=grads2["a"], adam_gb2=grads2["b"], adam_a2=params["a"], adam_b2=params["b"],
                        plr=np.array([position_lr(i, 5e-4, 5e-6, 1000) for i in (0, 250, 500, 1000, 2000)]))
    print("loss: ok")


def gen_scene_ops():
    """.3dcs checkpoints (sceneio.py:251-320) and densify_and_prune
    (density.py:54-105) known answers on float32-quantised scenes."""
    from convexsplat.density import densify_and_prune
    from convexsplat.sceneio import save_checkpoint
    from convexsplat.trainer import TrainConfig
    scene = quantize32(make_scene(9, seed=11, background=(0.1, 0.2, 0.3)))
    scene.scene_extent = 2.5
    for prec in (32, 16):
        save_checkpoint(os.path.join(OUT, f"ckpt_f{prec}.3dcs"), scene, precision=prec)
    arr = scene_arrays(scene)
    np.savez_compressed(os.path.join(OUT, "ckpt.npz"), **arr, scene_extent=scene.scene_extent)
    # densification: a scene with splits, low-opacity / low-mask / oversized convexes
    rng = np.random.default_rng(21)
    dscene = quantize32(make_scene(40, seed=12))
    dscene.scene_extent = 2.0
    prims = dscene.primitives
    prims[3].raw_opacity = float(np.float32(inverse_opacity_activation(0.02)))       # pruned: opacity
    prims[7].raw_mask = float(np.float32(inverse_mask_activation(0.005)))            # pruned: mask gate
    prims[11].points = (prims[11].points * 8.0).astype(np.float32).astype(np.float64)  # pruned: diameter
    prims[5].raw_opacity = float(np.float32(inverse_opacity_activation(0.035)))      # children pruned (0.8 o)
    signal = rng.uniform(0.0, 8e-6, size=len(prims)).astype(np.float32).astype(np.float64)
    signal[[3, 5, 11]] = 9e-6
    cfg = TrainConfig()
    before = scene_arrays(dscene)
    out = {}
    for tag, it in (("split", 600), ("nosplit", cfg.densify_stop + 1)):
        work = dscene.copy()
        work.scene_extent = dscene.scene_extent
        index_map, stats = densify_and_prune(work, signal, cfg, it)
        after = scene_arrays(work)
        for kk in ("points", "raw_delta", "raw_sigma", "raw_opacity", "raw_mask", "sh"):
            out[f"{tag}_{kk}"] = after[kk]
        out[f"{tag}_index_map"] = index_map
        out[f"{tag}_stats"] = np.array([stats.split, stats.pruned, stats.before, stats.after])
        out[f"{tag}_iteration"] = np.array(it)
    np.savez_compressed(os.path.join(OUT, "density.npz"), **{f"in_{k}": v for k, v in before.items()},
                        signal=signal, scene_extent=dscene.scene_extent, **out)
    print("scene ops: ok")


def main():
    DEPTH, NONE = ScalingMode.DEPTH, ScalingMode.NONE
    gen_scene_ops()
    gen_hulls()
    gen_loss()

    # config 1 of BASELINE.json: 1k convexes, 256^2, fwd+bwd
    s1 = make_scene(1000, 6, seed=0, spread=1.0)
    c1 = ring_cameras(1, size=256)[0]
    record("config1", s1, c1, DEPTH, RenderSettings(),
           d_image=loss_d_image(s1, c1, DEPTH, RenderSettings()))

    # exact settings vs the brute-force oracle (test_rasterize.py:118-128)
    s2 = make_scene(7, seed=10)
    c2 = ring_cameras(4, size=64)[0]
    rng = np.random.default_rng(2)
    record("exact7", s2, c2, DEPTH, EXACT_SETTINGS,
           d_image=rng.normal(0, 1e-3, size=(64, 64, 3)), reference=True)

    # scaling modes + sh degrees on a ragged (non multiple of 16) frame
    s3 = make_scene(40, seed=3, background=(0.2, 0.3, 0.1))
    base = ring_cameras(5, size=96)[2]
    c3 = Camera(fx=base.fx, fy=base.fy * 1.1, cx=50.0, cy=35.5, width=100, height=70,
                R=base.R, t=base.t)
    for mode, deg in ((ScalingMode.NONE, 0), (ScalingMode.SQRT_DEPTH, 1),
                      (ScalingMode.DEPTH, 2), (ScalingMode.DEPTH_SQUARED, 3)):
        st = RenderSettings(sh_degree=deg)
        rng = np.random.default_rng(3 + deg)
        record(f"mode_{MODE_NAME[mode]}", s3, c3, mode, st,
               d_image=rng.normal(0, 1e-2, size=(70, 100, 3)))

    # orthographic hexagons with saturated interiors (test_rasterize.py:30-84)
    hexes = Scene([hexagon((24.5, 24.5), 3.0, 0.5, (0.0, 1.0, 0.0)),
                   hexagon((24.5, 24.5), 2.0, 0.5, (1.0, 0.0, 0.0)),
                   hexagon((10.0, 30.0), 2.0, 0.7, (0.2, 0.2, 0.9), radius=6.0, sigma=0.8),
                   hexagon((40.0, 8.0), 2.5, 0.9, (0.9, 0.9, 0.1), radius=9.0, sigma=0.3, delta=0.5)],
                  background=np.array([0.1, 0.1, 0.1]))
    cam_o = ortho_camera(48)
    rng = np.random.default_rng(4)
    record("ortho_hex", hexes, cam_o, NONE, RenderSettings(),
           d_image=rng.normal(size=(48, 48, 3)))

    # K=7 with an interior point (test_backward.py:103-117)
    hx = hexagon((24.5, 24.5), 2.0, 0.6, (0.8, 0.3, 0.1))
    hx.points = np.vstack([hx.points, [[24.5, 24.5, 2.0]]])
    rng = np.random.default_rng(0)
    record("k7_interior", Scene([hx], background=np.zeros(3)), cam_o, NONE,
           RenderSettings(sh_degree=0), d_image=rng.normal(size=(48, 48, 3)))

    # culling: masked, behind camera, straddling the near plane, off-screen
    cull = [hexagon((24.5, 24.5), 2.0, 0.9, (1, 0, 0)), hexagon((24.5, 24.5), -2.0, 0.9, (0, 1, 0)),
            hexagon((24.5, 24.5), 2.0, 0.9, (0, 0, 1)), hexagon((500.0, 500.0), 2.0, 0.9, (1, 1, 0)),
            hexagon((20.0, 20.0), 1.5, 0.4, (0, 1, 1), radius=5.0)]
    cull[0].raw_mask = inverse_mask_activation(0.005)
    cull[2].points[0, 2] = 0.01
    record("culling", Scene(cull, background=np.array([0.3, 0.3, 0.3])), cam_o, NONE,
           RenderSettings(), d_image=np.ones((48, 48, 3)))

    # ALPHA_MAX cap (test_rasterize.py:188-194)
    cap = hexagon((24.5, 24.5), 2.0, 0.5, (1, 1, 1))
    cap.raw_opacity = 40.0
    record("alpha_cap", Scene([cap], background=np.zeros(3)), cam_o, NONE, RenderSettings(),
           d_image=np.full((48, 48, 3), 0.25))

    # equal depth: tie broken by scene index (test_rasterize.py:98-105)
    tie = Scene([hexagon((24.5, 24.5), 2.0, 0.5, (1, 0, 0)), hexagon((24.5, 24.5), 2.0, 0.5, (0, 1, 0))],
                background=np.zeros(3))
    record("depth_tie", tie, cam_o, NONE, RenderSettings(), d_image=np.ones((48, 48, 3)))

    # empty scene
    record("empty", Scene([], background=np.array([0.2, 0.4, 0.6])), cam_o, NONE, RenderSettings())

    # a denser perspective scene with many overlaps (production settings)
    s4 = make_scene(300, seed=11, spread=0.8)
    c4 = ring_cameras(3, size=128)[1]
    record("dense300", s4, c4, DEPTH, RenderSettings(),
           d_image=loss_d_image(s4, c4, DEPTH, RenderSettings(), seed=5))


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "loss":
        gen_loss()
    elif len(sys.argv) > 1 and sys.argv[1] == "scene_ops":
        gen_scene_ops()
    else:
        main()
