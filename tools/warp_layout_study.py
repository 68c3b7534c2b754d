"""Offline study: SIMT efficiency / MUFU work of blend thread layouts, from
the exact per-(pixel, candidate) evaluation sets of the CPU oracle on the
benchmark workload (sampled tiles).  Tooling only."""
import ctypes
import sys
import numpy as np

sys.path.insert(0, ".")
import oracle
from paper_2411_14974_b200 import synthetic

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
W, H = 1920, 1080
arrays = synthetic.quantize32(synthetic.generate_scene(n, 0))
cam = synthetic.bench_camera(W, H)
cam_d = synthetic.camera_dict(cam)
st = dict(cutoff=2e-4, floor=1e-4, tile=16, sh_degree=3, mode="depth", background=np.zeros(3))
view = oracle.prepare_view(arrays, cam_d, st, n_threads=8)
off, items = oracle.bin_tiles(view, W, H, 16)
T = off.size - 1
rng = np.random.default_rng(0)
tl = np.sort(rng.choice(T, size=min(T, 600), replace=False)).astype(np.int64)
tot = int(sum(off[t + 1] - off[t] for t in tl))
masks = np.zeros((tot, 8), np.uint32)
L = oracle.lib()
L.or_eval_masks.restype = ctypes.c_int64
L.or_eval_masks.argtypes = [ctypes.POINTER(oracle._Camera), ctypes.POINTER(oracle._Settings),
                            ctypes.POINTER(oracle._View), oracle._lp, oracle._ip, oracle._lp, ctypes.c_int64,
                            ctypes.POINTER(ctypes.c_uint32)]
c, s = oracle.make_camera(cam_d), oracle.make_settings(st)
L.or_eval_masks(ctypes.byref(c), ctypes.byref(s), ctypes.byref(view["_struct"]), off.ctypes.data_as(oracle._lp),
                items.ctypes.data_as(oracle._ip), tl.ctypes.data_as(oracle._lp), tl.size,
                masks.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32)))
bits = np.unpackbits(masks.view(np.uint8), bitorder="little").reshape(tot, 256).astype(bool)  # bit p = ly*16+lx
grid = bits.reshape(tot, 16, 16)  # [cand, ly, lx]
nl = view["hull_n"][view["order"][items[np.concatenate([np.arange(off[t], off[t + 1]) for t in tl])]]]
evals = bits.sum()
print(f"sample: {tl.size} tiles, {tot} (tile,candidate) pairs, {evals} pixel evals ({evals / (tl.size * 256):.1f}/px)")


def layout(wx, wy, px, py):
    """warps cover wx*wy pixels, each thread px*py pixels; returns warp-evals,
    thread-evals (threads with >=1 active pixel), pixel-evals inside active threads."""
    g = grid.reshape(tot, 16 // wy, wy, 16 // wx, wx)
    warp_active = g.any(axis=(2, 4))                      # [cand, nwy, nwx]
    t = grid.reshape(tot, 16 // py, py, 16 // px, px).any(axis=(2, 4))
    return int(warp_active.sum()), int(t.sum()), warp_active


for name, wx, wy, px, py in (("1px 8x4 warps", 8, 4, 1, 1), ("1px 16x2 warps", 16, 2, 1, 1),
                             ("1px 4x8 warps", 4, 8, 1, 1), ("2px(1x2) 8x8 warps", 8, 8, 2, 1),
                             ("2px(2x1) 8x8 warps", 8, 8, 1, 2), ("4px(2x2) 16x8", 16, 8, 2, 2),
                             ("4px(2x2) 8x16", 8, 16, 2, 2)):
    we, te, wa = layout(wx, wy, px, py)
    ppt = px * py
    lanes = we * 32
    # MUFU per warp-eval: base pixel nl+3, every further pixel of the thread 3 (incremental exp)
    nl_w = (wa.reshape(tot, -1).sum(axis=1) * nl).sum() / max(wa.sum(), 1)
    mufu = we * ((nl_w + 3) + 3 * (ppt - 1))
    print(f"{name:22s} warp-evals {we:9d}  SIMT eff {evals / (lanes * ppt):.3f}  thread-eff {te / lanes:.3f}"
          f"  MUFU warp-instr {mufu / 1e6:7.2f}M  (x{mufu / (evals / 32 * (nl_w + 3)):.2f} ideal)")

# "own list" layout: every lane walks its own pixel's candidates of a stage
# (kStageCands consecutive list entries) in order; a warp-stage costs
# max-over-lanes rounds.  Efficiency = pixel evals / (32 * rounds).
starts = np.concatenate([[0], np.cumsum([off[t + 1] - off[t] for t in tl])])
for stage in (16, 32, 64):
    rounds = 0
    cand_iters = 0
    for ti in range(tl.size):
        g = grid[starts[ti]:starts[ti + 1]]                  # [cand, 16, 16]
        blocks = g.reshape(-1, 4, 4, 2, 8).transpose(0, 1, 3, 2, 4).reshape(-1, 8, 32)  # [cand, warp, lane]
        for s0 in range(0, blocks.shape[0], stage):
            st_ = blocks[s0:s0 + stage]                      # [c, warp, lane]
            per_lane = st_.sum(axis=0)                       # [warp, lane]
            rounds += int(per_lane.max(axis=1).sum())
            cand_iters += int(st_.any(axis=2).sum())         # current scheme: candidates per warp
    print(f"own-list, stage {stage:3d}: SIMT eff {evals / (32 * rounds):.3f}  rounds {rounds}  "
          f"(per-candidate scheme: {cand_iters} warp-evals, eff {evals / (32 * cand_iters):.3f})")
