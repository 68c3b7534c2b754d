"""Scaling-mode parity diagnostics at 20k @640x480: image vs unforced and
forced oracle, count flips, per-kind gradient errors."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import paper_2411_14974_b200 as cs
from paper_2411_14974_b200 import rasterizer as rz, synthetic
import oracle
import test_gpu_parity as T

n, width, height = 20000, 640, 480
arrays = synthetic.quantize32(synthetic.generate_scene(n, seed=7))
cam = synthetic.bench_camera(width, height)
import os
MODES = [m for m in (("none", cs.ScalingMode.NONE), ("sqrt", cs.ScalingMode.SQRT_DEPTH),
                     ("depth", cs.ScalingMode.DEPTH), ("depth2", cs.ScalingMode.DEPTH_SQUARED))
         if m[0] in os.environ.get("MODES", "none,sqrt,depth,depth2").split(",")]
for mode, smode in MODES:
    st = cs.SceneTensors.from_arrays(arrays, "cuda")
    fr = rz.default_rasterizer().forward(st, cam, smode, cs.RenderSettings())
    o_set = dict(cutoff=2e-4, floor=1e-4, tile=16, sh_degree=3, mode=mode, background=np.zeros(3))
    cam_d = synthetic.camera_dict(cam)
    view = oracle.prepare_view(arrays, cam_d, o_set, n_threads=8)
    off, items = oracle.bin_tiles(view, width, height, 16)
    ref = oracle.render(arrays, cam_d, o_set, n_threads=8, view=view, tiles=(off, items))
    img = fr.image.cpu().numpy()
    dimg = np.abs(img - ref["image"])
    flips = int(np.sum(fr.count.cpu().numpy() != ref["count"]))
    forced_err = None
    try:
        forced = T.check_frame_forced(fr, arrays, cam_d, o_set, view, (off, items))
        forced_err = "ok"
    except AssertionError as e:
        forced = None
        forced_err = str(e)[:200]
    print(f"{mode}: unforced image max {dimg.max():.2e} at {np.unravel_index(dimg.argmax(), dimg.shape)}, flips {flips}, forced: {forced_err}")
    if forced is not None:
        d_img = np.random.default_rng(11).normal(0, 1e-2, size=(height, width, 3))
        grads = rz.default_rasterizer().backward(fr, torch.tensor(d_img, dtype=torch.float32), rz.zero_grads(st))
        og, _ = T.record_and_force(fr, arrays, cam_d, o_set, d_img, view, (off, items), forced=forced)
        g = {k: v.cpu().numpy() for k, v in grads.items()}
        print("   ", {k: f"{v:.2e}" for k, v in T.kind_errors(g, og, n, T.GRAD_FLOOR).items()})
        # the worst raw_delta entries
        a, b = g["raw_delta"].ravel(), np.asarray(og["d_raw_delta"]).ravel()
        fl = max(T.GRAD_FLOOR * np.abs(b).max(), 1e-12)
        rel = np.abs(a - b) / np.maximum(np.maximum(np.abs(a), np.abs(b)), fl)
        w = np.argsort(rel)[-3:]
        print("    worst raw_delta:", [(int(i), float(a[i]), float(b[i]), float(rel[i])) for i in w], "max", float(np.abs(b).max()))
