import torch, paper_2411_14974_b200 as cs
from paper_2411_14974_b200 import synthetic
arrays = synthetic.quantize32(synthetic.generate_scene(3000, seed=4))
st = cs.SceneTensors.from_arrays(arrays, "cuda")
cam = synthetic.ring_cameras(1, 96, 72)[0]
out = cs.render(st, cam)
print("ok", out.image.mean())
