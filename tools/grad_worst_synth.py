"""Worst packed-gradient entries (floor 2e-4 x max) of the GPU backward vs the C oracle on a synthetic scene."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import oracle
import paper_2411_14974_b200 as cs
from paper_2411_14974_b200 import rasterizer as rz, synthetic

n, w, h, seed = (int(v) for v in (sys.argv[1:5] if len(sys.argv) > 4 else (20000, 640, 480, 1)))
dseed = int(sys.argv[5]) if len(sys.argv) > 5 else seed   # upstream-gradient seed
arrays = synthetic.quantize32(synthetic.generate_scene(n, seed))
cam = synthetic.bench_camera(w, h)
st = cs.SceneTensors.from_arrays(arrays, "cuda")
fr = rz.default_rasterizer().forward(st, cam, cs.ScalingMode.DEPTH, cs.RenderSettings())
o_set = dict(cutoff=2e-4, floor=1e-4, tile=16, sh_degree=3, mode="depth", background=np.zeros(3))
cam_d = synthetic.camera_dict(cam)
view = oracle.prepare_view(arrays, cam_d, o_set, n_threads=16)
off, items = oracle.bin_tiles(view, w, h, 16)
d_img = np.random.default_rng(dseed).normal(0, 1e-2, size=(h, w, 3))
grads = rz.default_rasterizer().backward(fr, torch.tensor(d_img, dtype=torch.float32), rz.zero_grads(st))
og = oracle.backward(arrays, cam_d, o_set, d_img, n_threads=16, view=view, tiles=(off, items))
kinds = (("points", "d_points"), ("raw_delta", "d_raw_delta"), ("raw_sigma", "d_raw_sigma"),
         ("raw_opacity", "d_raw_opacity"), ("sh", "d_sh"), ("raw_mask", "d_raw_mask"))
A = np.concatenate([grads[a].cpu().numpy().reshape(n, -1) for a, _ in kinds], 1)
B = np.concatenate([og[b].reshape(n, -1) for _, b in kinds], 1)
labels = np.concatenate([np.array([f"{a}[{j}]" for j in range(grads[a].reshape(n, -1).shape[1])]) for a, _ in kinds])
den = np.maximum(np.abs(A), np.abs(B))
m = den.max()
rel = np.abs(A - B) / np.maximum(den, 2e-4 * m)
for idx in np.argsort(rel.ravel())[::-1][:12]:
    i, j = np.unravel_index(idx, rel.shape)
    print(f"convex {i:5d} {labels[j]:16s} rel {rel[i, j]:.2e} gpu {A[i, j]: .5e} ref {B[i, j]: .5e} |ref|/max {abs(B[i, j]) / m:.1e}")
i = int(np.unravel_index(np.argmax(rel), rel.shape)[0])
print("worst convex points grad gpu\n", A[i, :18].reshape(6, 3), "\nref\n", B[i, :18].reshape(6, 3))
