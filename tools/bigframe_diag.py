"""Gradient-error anatomy on a large frame (131k tiles): flips, run-to-run
atomic noise, and the per-field / per-convex error distribution against the
float64 oracle."""
import sys
import numpy as np
import torch

sys.path.insert(0, ".")
import oracle
import paper_2411_14974_b200 as cs
from paper_2411_14974_b200 import rasterizer as rz, synthetic
from tests.test_gpu_parity import GRAD_KINDS, GRAD_FLOOR, pack, packed_error

n, w, h, seed = (int(a) for a in (sys.argv[1:5] if len(sys.argv) > 4 else (4000, 8208, 4112, 3)))
arrays = synthetic.quantize32(synthetic.generate_scene(n, seed))
cam = synthetic.bench_camera(w, h)
st = cs.SceneTensors.from_arrays(arrays, "cuda")
r = rz.default_rasterizer()
fr = r.forward(st, cam, cs.ScalingMode.DEPTH, cs.RenderSettings())
info = rz.inspect_frame(fr)
o_set = dict(cutoff=2e-4, floor=1e-4, tile=16, sh_degree=3, mode="depth", background=np.zeros(3))
cam_d = synthetic.camera_dict(cam)
view = oracle.prepare_view(arrays, cam_d, o_set, n_threads=16)
off, items = oracle.bin_tiles(view, w, h, 16)
ref = oracle.render(arrays, cam_d, o_set, n_threads=16, view=view, tiles=(off, items))
count = fr.count.cpu().numpy()
flips = np.argwhere(count != ref["count"])
print("pairs", items.size, "flipped pixels", len(flips), "img err", np.abs(fr.image.cpu().numpy() - ref["image"]).max())
rng = np.random.default_rng(seed)
d_img = rng.normal(0, 1e-2, size=(h, w, 3))
dt = torch.tensor(d_img, dtype=torch.float32)
g1 = r.backward(fr, dt, rz.zero_grads(st))
g2 = r.backward(fr, dt, rz.zero_grads(st))
og = oracle.backward(arrays, cam_d, o_set, d_img, n_threads=16, view=view, tiles=(off, items))
bb = info["bbox"]
keep = np.ones(n, bool)
for y, x in flips:
    keep &= ~((bb[:, 0] <= x) & (x < bb[:, 1]) & (bb[:, 2] <= y) & (y < bb[:, 3]))
area = (bb[:, 1] - bb[:, 0]).clip(0) * (bb[:, 3] - bb[:, 2]).clip(0)
print("kept convexes", keep.sum(), "median bbox px", int(np.median(area)), "max", int(area.max()))
for kind in GRAD_KINDS:
    a = g1[kind[2]].cpu().numpy().reshape(n, -1)
    b = g2[kind[2]].cpu().numpy().reshape(n, -1)
    o = np.asarray(og[kind[3]]).reshape(n, -1)
    print(f"{kind[2]:>14}: vs oracle {packed_error(a.ravel(), o.ravel(), GRAD_FLOOR):.2e} "
          f"(no-flip {packed_error(a[keep].ravel(), o[keep].ravel(), GRAD_FLOOR):.2e}), run-to-run "
          f"{packed_error(a.ravel(), b.ravel(), GRAD_FLOOR):.2e}")
ours = pack({k: v.cpu().numpy() for k, v in g1.items()}, [k[2] for k in GRAD_KINDS], n).reshape(n, -1)
theirs = pack(og, [k[3] for k in GRAD_KINDS], n).reshape(n, -1)
denom = np.maximum(np.abs(ours), np.abs(theirs))
rel = np.abs(ours - theirs) / np.maximum(denom, GRAD_FLOOR * denom.max())
worst = np.argsort(rel.max(1))[::-1][:8]
for i in worst:
    j = int(rel[i].argmax())
    print(f"convex {i}: rel {rel[i].max():.2e} col {j} ours {ours[i, j]:.4e} ref {theirs[i, j]:.4e} "
          f"bbox px {area[i]} kept {keep[i]} bbox {bb[i]}")
relk = rel[keep].ravel()
print(f"no-flip: max {relk.max():.2e} 99.99% {np.quantile(relk, 0.9999):.2e} 99.9% {np.quantile(relk, 0.999):.2e}")
