"""Forward blend consumer wait breakdown (library built with -DCS_WAIT_STATS)."""
import sys
sys.path.insert(0, ".")
import torch
import paper_2411_14974_b200 as cs
from paper_2411_14974_b200 import rasterizer as rz, synthetic
arrays = synthetic.quantize32(synthetic.generate_scene(1_000_000, 0))
st = cs.SceneTensors.from_arrays(arrays, "cuda")
cam = synthetic.bench_camera(1920, 1080)
r = rz.default_rasterizer()
fr = r.forward(st, cam)
r.launch_forward(fr, 0, 1)
fr.workspace.counters()[32:40].zero_()
r.launch_forward(fr, 2, 2)
c = fr.workspace.counters().cpu()[32:40].view(torch.int64).tolist()
first, rest, done, total = c
print(f"consumer-warp cycles: total {total:.3e}; waiting for stage data: first batch {first / total:.1%}, "
      f"later batches (warp busy) {rest / total:.1%}, after the warp finished its pixels {done / total:.1%}")
