"""Fraction of blend-kernel time spent waiting in the producer/consumer
pipeline (library built with -DCS_WAIT_STATS, e.g.
bash tools/build_variant.sh ws -DCS_WAIT_STATS blend; CS_LIB_PATH=variants/ws.so)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2411_14974_b200 as cs  # noqa: E402
from paper_2411_14974_b200 import _lib, rasterizer as rz, synthetic  # noqa: E402

n, w, h = 1_000_000, 1920, 1080
arrays = synthetic.quantize32(synthetic.generate_scene(n, 0))
cam = synthetic.bench_camera(w, h)
st = cs.SceneTensors.from_arrays(arrays, "cuda")
r = rz.Rasterizer("cuda")
fr = r.forward(st, cam, cs.ScalingMode.DEPTH, cs.RenderSettings())
d = torch.randn(h, w, 3, device="cuda") * 1e-3
grads = rz.zero_grads(st)
L = _lib.load()
buf = (ctypes.c_ulonglong * 12)()
L.cs_debug_wait_stats(buf, 1)
r.launch_forward(fr, 2, 2)
r.launch_backward(fr, d, grads, 0, 0)
L.cs_debug_wait_stats(buf, 0)
v = list(buf)
print(f"forward : consumers wait on full {100 * v[1] / max(v[0], 1):.1f}% of their cycles; "
      f"producer waits on empty {100 * v[3] / max(v[2], 1):.1f}% of its cycles; "
      f"first-batch waits {100 * v[8] / max(v[0], 1):.1f}%")
print(f"backward: consumers wait on full {100 * v[5] / max(v[4], 1):.1f}% of their cycles; "
      f"producer waits on empty {100 * v[7] / max(v[6], 1):.1f}% of its cycles")
