"""Gradient parity at the GPU's own discrete decisions (diagnostics).

For each case: GPU forward + backward through the C ABI, the GPU's blend
decisions (cs_forward_record), the float64 oracle backward forced to those
decisions, then per parameter kind the reference's relative error
|a-b| / max(|a|, |b|, floor) with floor = max(1e-6 * max_kind, 1e-12)
(backward.py:464-467, applied per kind).  Also prints the unforced figure.

    python tools/grad_forced.py [case ...]     (cases: see CASES below)
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import paper_2411_14974_b200 as cs  # noqa: E402
from paper_2411_14974_b200 import rasterizer as rz, synthetic  # noqa: E402
from tests import golden_cases as gc  # noqa: E402

KINDS = (("points", "d_points"), ("raw_delta", "d_raw_delta"), ("raw_sigma", "d_raw_sigma"),
         ("raw_opacity", "d_raw_opacity"), ("sh", "d_sh"), ("raw_mask", "d_raw_mask"))


def per_kind(gpu, ref, n):
    out = {}
    for a_name, b_name in KINDS:
        a = gpu[a_name].reshape(n, -1).astype(np.float64)
        b = ref[b_name].reshape(n, -1)
        den = np.maximum(np.abs(a), np.abs(b))
        if den.size == 0 or den.max() == 0:
            out[a_name] = (0.0, "")
            continue
        floor = max(1e-6 * den.max(), 1e-12)
        rel = np.abs(a - b) / np.maximum(den, floor)
        i = np.unravel_index(int(np.argmax(rel)), rel.shape)
        out[a_name] = (float(rel.max()), f"convex {i[0]} [{i[1]}] gpu={a[i]:.6e} ref={b[i]:.6e} "
                                         f"|ref|/max={abs(b[i]) / den.max():.1e} q9999={np.quantile(rel, 0.9999):.1e}")
    return out


def run(name, arrays, cam, mode, settings, d_img, n_threads=16):
    st = cs.SceneTensors.from_arrays(arrays, "cuda", background=arrays.get("background"))
    r = rz.default_rasterizer()
    fr = r.forward(st, cam, mode, settings)
    grads = r.backward(fr, torch.tensor(d_img, dtype=torch.float32), rz.zero_grads(st))
    gpu = {k: v.cpu().numpy() for k, v in grads.items()}
    offsets, pos, clamp = rz.record_blends(fr)
    o_set = dict(cutoff=settings.contribution_cutoff, floor=settings.transmittance_floor, tile=16,
                 sh_degree=settings.sh_degree, mode=mode.value,
                 background=np.asarray(arrays.get("background", np.zeros(3)), dtype=np.float64))
    cam_d = synthetic.camera_dict(cam)
    t0 = time.time()
    view = oracle.prepare_view(arrays, cam_d, o_set, n_threads=n_threads)
    tiles = oracle.bin_tiles(view, cam.width, cam.height, 16)
    own = oracle.blend_decisions(cam_d, o_set, view, tiles)
    flips = int(np.sum(np.diff(own[0]) != np.diff(offsets)))
    og = oracle.backward(arrays, cam_d, o_set, d_img, n_threads=n_threads, view=view, tiles=tiles,
                         forced=(offsets, pos, clamp))
    ou = oracle.backward(arrays, cam_d, o_set, d_img, n_threads=n_threads, view=view, tiles=tiles)
    n = st.n
    f = per_kind(gpu, og, n)
    u = per_kind(gpu, ou, n)
    print(f"== {name}: n={n} {cam.width}x{cam.height} blends={int(offsets[-1])} count-flipped pixels={flips} "
          f"(oracle {time.time() - t0:.1f}s)")
    for k, _ in KINDS:
        print(f"   {k:12s} forced {f[k][0]:.2e} | unforced {u[k][0]:.2e}   {f[k][1]}")
    return max(v[0] for v in f.values())


def golden(name):
    g = gc.load(name)
    c, s_ = gc.camera(g), gc.settings(g)
    cam = cs.Camera(fx=c["fx"], fy=c["fy"], cx=c["cx"], cy=c["cy"], width=c["width"], height=c["height"],
                    R=c["R"], t=c["t"], z_near=c["z_near"], ortho=c["ortho"])
    settings = cs.RenderSettings(contribution_cutoff=s_["cutoff"], transmittance_floor=s_["floor"],
                                 tile_size=s_["tile"], sh_degree=s_["sh_degree"])
    arrays = dict(gc.params(g), background=g["background"])
    return arrays, cam, cs.ScalingMode(s_["mode"]), settings, g["d_image"]


def synth(n, w, h, seed, k=6, exact=False, ortho=False):
    arrays = synthetic.quantize32(synthetic.generate_scene(n, seed, k=k) if k != 6 else synthetic.generate_scene(n, seed))
    if ortho:
        cam = cs.Camera(fx=40.0, fy=40.0, cx=w / 2, cy=h / 2, width=w, height=h, R=np.eye(3),
                        t=np.array([0.0, 0.0, 4.0]), ortho=True)
    else:
        cam = synthetic.bench_camera(w, h)
    settings = cs.EXACT_SETTINGS if exact else cs.RenderSettings()
    d_img = np.random.default_rng(seed).normal(0, 1e-2, size=(h, w, 3))
    return arrays, cam, cs.ScalingMode.DEPTH, settings, d_img


CASES = {
    "2k": lambda: synth(2000, 320, 200, 0),
    "20k": lambda: synth(20000, 640, 480, 1),
    "exact": lambda: synth(400, 128, 96, 21, exact=True),
    "ortho": lambda: synth(400, 128, 96, 21, ortho=True),
    "k12": lambda: synth(1500, 200, 136, 12, k=12),
    "131k_tiles": lambda: synth(4000, 8208, 4112, 3),
    "max_width": lambda: synth(3000, 32767, 40, 4),
    "100k": lambda: synth(100_000, 1297, 840, 0),
    "1M": lambda: synth(1_000_000, 1920, 1080, 0),
}

if __name__ == "__main__":
    names = sys.argv[1:] or (["golden"] + [c for c in CASES if c not in ("1M",)])
    worst = 0.0
    for nm in names:
        if nm == "golden":
            for gname in gc.scene_cases():
                g = gc.load(gname)
                if "d_image" in g:
                    worst = max(worst, run(gname, *golden(gname)))
        else:
            worst = max(worst, run(nm, *CASES[nm]()))
    print(f"WORST forced per-kind error: {worst:.2e}")
