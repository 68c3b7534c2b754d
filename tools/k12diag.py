import sys, numpy as np, torch
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import paper_2411_14974_b200 as cs
from paper_2411_14974_b200 import rasterizer as rz, synthetic
import oracle, test_gpu_parity as T
k, mode = 12, "none"
n, width, height = 1500, 200, 136
arrays = synthetic.quantize32(synthetic.generate_scene(n, seed=k, k=k))
cam = synthetic.bench_camera(width, height)
st = cs.SceneTensors.from_arrays(arrays, "cuda")
fr = rz.default_rasterizer().forward(st, cam, cs.ScalingMode.NONE, cs.RenderSettings())
o_set = dict(cutoff=2e-4, floor=1e-4, tile=16, sh_degree=3, mode=mode, background=np.zeros(3))
cam_d = synthetic.camera_dict(cam)
view = oracle.prepare_view(arrays, cam_d, o_set, n_threads=8)
off, items = oracle.bin_tiles(view, width, height, 16)
forced = T.check_frame_forced(fr, arrays, cam_d, o_set, view, (off, items))
d_img = np.random.default_rng(k).normal(0, 1e-2, size=(height, width, 3))
grads = rz.default_rasterizer().backward(fr, torch.tensor(d_img, dtype=torch.float32), rz.zero_grads(st))
og, _ = T.record_and_force(fr, arrays, cam_d, o_set, d_img, view, (off, items), forced=forced)
a = grads["points"].cpu().numpy().reshape(n, -1).astype(np.float64); b = np.asarray(og["d_points"]).reshape(n, -1)
den = np.maximum(np.abs(a), np.abs(b)); fl = 5e-4 * den.max()
r = np.abs(a - b) / np.maximum(den, fl)
idx = np.unravel_index(np.argsort(r.ravel())[-5:], r.shape)
for i, j in zip(*idx):
    print(f"convex {i} comp {j}: gpu {a[i,j]:.6e} ref {b[i,j]:.6e} rel {r[i,j]:.2e}  |entry|/max {den[i,j]/den.max():.2e}  hull_n {view['hull_n'][i]} bbox {view['bbox'][i]} delta_s {view['delta_s'][i]:.3g} sigma_s {view['sigma_s'][i]:.3g}")
print("max_kind", den.max())
