import sys; sys.path.insert(0, ".")
import numpy as np, torch
import oracle
import paper_2411_14974_b200 as cs
from paper_2411_14974_b200 import rasterizer as rz, synthetic
n, w, h = 1000000, 1920, 1080
arrays = synthetic.quantize32(synthetic.generate_scene(n, 0))
cam = synthetic.bench_camera(w, h)
st = cs.SceneTensors.from_arrays(arrays, "cuda")
fr = rz.default_rasterizer().forward(st, cam, cs.ScalingMode.DEPTH, cs.RenderSettings())
o_set = dict(cutoff=2e-4, floor=1e-4, tile=16, sh_degree=3, mode="depth", background=np.zeros(3))
cam_d = synthetic.camera_dict(cam)
view = oracle.prepare_view(arrays, cam_d, o_set, n_threads=16)
off, items = oracle.bin_tiles(view, w, h, 16)
ref = oracle.render(arrays, cam_d, o_set, n_threads=16, view=view, tiles=(off, items))
cg = fr.count.cpu().numpy(); co = ref["count"]
d = np.argwhere(cg != co)
print("pixels with different blend counts:", len(d))
for y, x in d[:10]:
    print(y, x, cg[y, x], co[y, x], "T gpu", float(fr.final_T[y, x]), "T ref", ref["trans"][y, x])
b = np.asarray(rz.inspect_frame(fr)["bbox"][630767])
print("bbox of 630767", b)
for y, x in d:
    if b[0] <= x < b[1] and b[2] <= y < b[3]: print("flip inside 630767 bbox at", y, x)
