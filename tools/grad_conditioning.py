"""Conditioning of the reference gradients under float32 input rounding (CPU).

The float64 oracle's backward at its own blend decisions, recomputed after
rounding ONLY the per-convex values the GPU keeps in float32 (colour,
opacity, sigma_s, delta_s) and the upstream gradient d_image to float32:
the relative change of each gradient kind (floor 2e-4 x max_kind) is the
error any float32 implementation inherits from its inputs alone, before a
single float32 operation.

    python tools/grad_conditioning.py [mode] [seed]
"""
import numpy as np, sys
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
import oracle
from paper_2411_14974_b200 import synthetic
n, w, h = 20000, 640, 480
mode = sys.argv[1] if len(sys.argv) > 1 else "depth"
seed = int(sys.argv[2]) if len(sys.argv) > 2 else 1
arrays = synthetic.quantize32(synthetic.generate_scene(n, seed))
cam = synthetic.camera_dict(synthetic.bench_camera(w, h))
o_set = dict(cutoff=2e-4, floor=1e-4, tile=16, sh_degree=3, mode=mode, background=np.zeros(3))
d_img = np.random.default_rng(seed).normal(0, 1e-2, size=(h, w, 3))
def run(q_inputs, q_dimg):
    view = oracle.prepare_view(arrays, cam, o_set, n_threads=8)
    if q_inputs:
        for k in q_inputs:
            view[k][:] = view[k].astype(np.float32).astype(np.float64)
    tiles = oracle.bin_tiles(view, w, h, 16)
    forced = oracle.blend_decisions(cam, o_set, view, tiles)
    d = d_img.astype(np.float32).astype(np.float64) if q_dimg else d_img
    return oracle.backward(arrays, cam, o_set, d, n_threads=8, view=view, tiles=tiles, forced=forced)
base = run([], False)
def err(a, b, k):
    x, y = a[k].ravel(), b[k].ravel()
    den = np.maximum(np.abs(x), np.abs(y)); fl = 2e-4 * den.max()
    r = np.abs(x - y) / np.maximum(den, fl)
    i = int(np.argmax(r)); return f"{r.max():.1e} @{i}"
for label, qi, qd in [("d_image f32", [], True), ("colour f32", ["color"], False), ("opacity f32", ["opacity"], False),
                      ("sigma_s,delta_s f32", ["sigma_s", "delta_s"], False),
                      ("all", ["color", "opacity", "sigma_s", "delta_s"], True)]:
    g = run(qi, qd)
    print(label, {k: err(g, base, k) for k in ("d_raw_sigma", "d_raw_delta", "d_points", "d_raw_opacity", "d_sh")})
