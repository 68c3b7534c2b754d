"""Forward outputs of the current library vs a variant (CS_LIB_PATH in a
subprocess) on the 1M @1080p bench scene: exact equality expected when a
change only skips work.  usage: python tools/cull_check.py variants/x.so"""
import os
import subprocess
import sys

import numpy as np

code = r'''
import sys, numpy as np, torch
sys.path.insert(0, ".")
import paper_2411_14974_b200 as cs
from paper_2411_14974_b200 import synthetic, rasterizer as rz
arrays = synthetic.quantize32(synthetic.generate_scene(1_000_000, 0))
st = cs.SceneTensors.from_arrays(arrays, "cuda")
fr = rz.default_rasterizer().forward(st, synthetic.bench_camera(1920, 1080))
np.savez(sys.argv[1], image=fr.image.cpu().numpy(), count=fr.count.cpu().numpy(), T=fr.final_T.cpu().numpy())
'''
env = dict(os.environ)
subprocess.run([sys.executable, "-c", code, "/tmp/cull_a.npz"], check=True, env=env)
env["CS_LIB_PATH"] = sys.argv[1]
subprocess.run([sys.executable, "-c", code, "/tmp/cull_b.npz"], check=True, env=env)
a, b = np.load("/tmp/cull_a.npz"), np.load("/tmp/cull_b.npz")
for k in ("image", "count", "T"):
    print(k, "identical" if np.array_equal(a[k], b[k]) else f"DIFFERENT max {np.abs(a[k].astype(np.float64) - b[k]).max():.3e}, {int((a[k] != b[k]).sum())} entries")
