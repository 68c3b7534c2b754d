"""Per-tile load balance of the 8x4 warp blocks (blend counts as the work proxy), 1M @1080p."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2411_14974_b200 as cs
from paper_2411_14974_b200 import rasterizer as rz, synthetic

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
arrays = synthetic.generate_scene(n, 0)
st = cs.SceneTensors.from_arrays(synthetic.quantize32(arrays), "cuda")
cam = synthetic.bench_camera(1920, 1080)
fr = rz.default_rasterizer().forward(st, cam, cs.ScalingMode.DEPTH, cs.RenderSettings())
cnt = fr.count.cpu().numpy().astype(np.int64)
H, W = cnt.shape
Hp, Wp = (H + 15) // 16 * 16, (W + 15) // 16 * 16
c = np.zeros((Hp, Wp), np.int64)
c[:H, :W] = cnt
blk = c.reshape(Hp // 4, 4, Wp // 8, 8).sum(axis=(1, 3))          # 8x4 blocks
tiles = blk.reshape(Hp // 16, 4, Wp // 16, 2).transpose(0, 2, 1, 3).reshape(-1, 8)
busy = tiles.sum(1) > 0
mx, mean = tiles.max(1)[busy], tiles.mean(1)[busy]
print(f"tiles {busy.sum()}  sum(max)/sum(mean) = {mx.sum() / mean.sum():.3f}  (1.0 = balanced warps)")
# per-pixel maxima inside a warp (SIMT divergence proxy)
lane = c.reshape(Hp // 4, 4, Wp // 8, 8).max(axis=(1, 3))
print(f"sum(max over lanes)/sum(mean over lanes) per warp block = {lane.sum() / (blk.sum() / 32):.3f}")
