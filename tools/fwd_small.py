"""Small forward/backward through the C ABI (for compute-sanitizer runs)."""
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2411_14974_b200 as cs
from paper_2411_14974_b200 import rasterizer as rz, synthetic

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
w, h = (int(sys.argv[2]), int(sys.argv[3])) if len(sys.argv) > 3 else (320, 200)
mode = {"depth": cs.ScalingMode.DEPTH, "depth2": cs.ScalingMode.DEPTH_SQUARED, "none": cs.ScalingMode.NONE,
        "sqrt": cs.ScalingMode.SQRT_DEPTH}[sys.argv[4] if len(sys.argv) > 4 else "depth"]
arrays = synthetic.quantize32(synthetic.generate_scene(n, 0))
cam = synthetic.bench_camera(w, h)
st = cs.SceneTensors.from_arrays(arrays, "cuda")
r = rz.Rasterizer("cuda")
fr = r.forward(st, cam, mode, cs.RenderSettings())
g = r.backward(fr, torch.randn(h, w, 3) * 1e-2, rz.zero_grads(st))
torch.cuda.synchronize()
print("ok", fr.n_visible, fr.n_pairs, float(fr.image.sum()), float(g["points"].abs().sum()))
