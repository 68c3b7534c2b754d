"""Compare forward outputs, pixel_last and backward gradients of the current
library against a variant (CS_LIB_PATH in a subprocess).
usage: python tools/cmp_libs.py variants/x.so [n w h]"""
import os
import subprocess
import sys

import numpy as np

code = r'''
import sys, numpy as np, torch
sys.path.insert(0, ".")
import paper_2411_14974_b200 as cs
from paper_2411_14974_b200 import synthetic, rasterizer as rz
n, w, h = (int(v) for v in sys.argv[2:5])
arrays = synthetic.quantize32(synthetic.generate_scene(n, 1))
st = cs.SceneTensors.from_arrays(arrays, "cuda")
r = rz.default_rasterizer()
fr = r.forward(st, synthetic.bench_camera(w, h))
ws = fr.workspace
last = ws.region("pixel_last", torch.int32, w * h).cpu().numpy()
T = ws.region("pixel_T", torch.float32, w * h).cpu().numpy()
clamp = ws.region("pixel_clamp", torch.uint8, w * h).cpu().numpy()
L = ws.layout
tiles = L.tiles_x * L.tiles_y
# blend masks: 8 arrays of mask_words after the tile order in the scratch; compare the words the
# backward may read (tile t, batch b < its batch count)
ranges = ws.region("tile_ranges", torch.int32, 2 * tiles).cpu().numpy().reshape(tiles, 2).astype(np.int64)
off = L.scratch + ((4 * (1 << 17) + 255) // 256) * 256
cap_al = (L.pair_ids - L.pair_tiles) // 4
nw = ((cap_al * 4 + 255) // 256 * 256) // 4 // 32 + tiles + 2
raw = torch.empty(0, dtype=torch.uint8, device="cuda")
buf = ws.buffer[off:off + 8 * nw * 4].view(torch.int32).cpu().numpy().reshape(8, nw) if hasattr(ws, "buffer") else None
d = torch.tensor(np.random.default_rng(1).normal(0, 1e-2, size=(h, w, 3)), dtype=torch.float32)
g = r.backward(fr, d, rz.zero_grads(st))
sel = []
if buf is not None:
    for t in range(tiles):
        x0, x1 = ranges[t]
        nb = (x1 - x0 + 31) // 32 if x1 > x0 else 0
        for b in range(nb):
            sel.append((x0 >> 5) + t + b)
masks = buf[:, sel] if buf is not None else np.zeros(1)
np.savez(sys.argv[1], masks=masks, clamp=clamp, image=fr.image.cpu().numpy(), count=fr.count.cpu().numpy(), last=last, T=T,
         vis=fr.visible.cpu().numpy(), gp=g["points"].cpu().numpy(), go=g["raw_opacity"].cpu().numpy())
'''
args = sys.argv[2:5] if len(sys.argv) > 4 else ["20000", "640", "480"]
env = dict(os.environ)
env.pop("CS_LIB_PATH", None)
subprocess.run([sys.executable, "-c", code, "/tmp/cmp_a.npz", *args], check=True, env=env)
env["CS_LIB_PATH"] = sys.argv[1]
subprocess.run([sys.executable, "-c", code, "/tmp/cmp_b.npz", *args], check=True, env=env)
a, b = np.load("/tmp/cmp_a.npz"), np.load("/tmp/cmp_b.npz")
for k in a.files:
    x, y = a[k], b[k]
    diff = np.abs(x.astype(np.float64) - y.astype(np.float64))
    print(f"{k:6s} equal={np.array_equal(x, y)} max|diff|={diff.max():.3g} n_diff={(diff > 0).sum()}")
