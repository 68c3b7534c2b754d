"""Worst packed-gradient entries (floor 1e-4 x max) of the GPU backward vs a golden fixture."""
import sys
import numpy as np
sys.path.insert(0, ".")
from tests import golden_cases as gc
from tests.test_gpu_parity import make_objects
import paper_2411_14974_b200 as cs

name = sys.argv[1] if len(sys.argv) > 1 else "mode_none"
g = gc.load(name)
cam, settings, mode, st = make_objects(g)
gb = cs.backward(st, cam, g["d_image"], mode, settings)
n = g["points"].shape[0]
kinds = (("d_points", "g_points"), ("d_raw_delta", "g_delta"), ("d_raw_sigma", "g_sigma"),
         ("d_raw_opacity", "g_opacity"), ("d_sh", "g_sh"), ("d_raw_mask", "g_mask"))
A = np.concatenate([getattr(gb, a).reshape(n, -1) for a, _ in kinds], 1)
B = np.concatenate([g[b].reshape(n, -1) for _, b in kinds], 1)
labels = np.concatenate([np.array([f"{a}[{j}]" for j in range(getattr(gb, a).reshape(n, -1).shape[1])])
                         for a, _ in kinds])
den = np.maximum(np.abs(A), np.abs(B))
m = den.max()
rel = np.abs(A - B) / np.maximum(den, 1e-4 * m)
for idx in np.argsort(rel.ravel())[::-1][:12]:
    i, j = np.unravel_index(idx, rel.shape)
    print(f"convex {i:4d} {labels[j]:16s} rel {rel[i, j]:.2e} gpu {A[i, j]: .5e} ref {B[i, j]: .5e} |ref|/max {abs(B[i, j]) / m:.1e}")
