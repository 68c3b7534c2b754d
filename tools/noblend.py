import sys; sys.path.insert(0, ".")
import torch
import paper_2411_14974_b200 as cs
from paper_2411_14974_b200 import rasterizer as rz, synthetic
st = cs.SceneTensors.from_arrays(synthetic.quantize32(synthetic.generate_scene(1_000_000, 0)), "cuda")
r = rz.default_rasterizer()
fr = r.forward(st, synthetic.bench_camera(1920, 1080))
c = fr.workspace.counters().cpu()[16:32].view(torch.int64).tolist()
print("warp-evals", c[5], "without any blend", c[7], f"({c[7] / c[5]:.1%})", "lane evals", c[0], "blends", c[2])
