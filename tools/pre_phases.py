"""Preprocess time per phase (library built with -DCS_PRE_PHASES:
bash tools/build_variant_pre.sh ph -DCS_PRE_PHASES; CS_LIB_PATH=variants/ph.so).
usage: python tools/pre_phases.py [n w h]"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2411_14974_b200 as cs  # noqa: E402
from paper_2411_14974_b200 import _lib, rasterizer as rz, synthetic  # noqa: E402

n, w, h = (int(v) for v in sys.argv[1:4]) if len(sys.argv) > 3 else (1_000_000, 1920, 1080)
arrays = synthetic.quantize32(synthetic.generate_scene(n, 0))
st = cs.SceneTensors.from_arrays(arrays, "cuda")
r = rz.Rasterizer("cuda")
fr = r.forward(st, synthetic.bench_camera(w, h))
L = _lib.load()
buf = (ctypes.c_ulonglong * 8)()
L.cs_debug_pre_phases(buf, 1)
r.launch_forward(fr, 0, 0)
L.cs_debug_pre_phases(buf, 0)
names = ["mask gate + loads", "projection", "graham scan", "lines + bbox loop", "bbox + discrete writes",
         "colour + record"]
tot = sum(buf[:6])
for i, nm in enumerate(names):
    print(f"{nm:26s} {100 * buf[i] / tot:5.1f}%  ({buf[i] / max(n, 1):8.0f} cycles per convex)")
