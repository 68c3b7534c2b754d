"""Diagnostics: per-kind gradient error of the GPU backward vs the golden fixtures."""
import sys
import numpy as np
sys.path.insert(0, ".")
from tests import golden_cases as gc
from tests.test_gpu_parity import make_objects, grad_rel_error
import paper_2411_14974_b200 as cs

for name in sys.argv[1:] or ["mode_depth", "dense300", "config1", "ortho_hex", "k7_interior", "exact7"]:
    g = gc.load(name)
    cam, settings, mode, st = make_objects(g)
    gb = cs.backward(st, cam, g["d_image"], mode, settings)
    print(f"== {name}")
    for ours, theirs in (("d_points", "g_points"), ("d_raw_delta", "g_delta"), ("d_raw_sigma", "g_sigma"),
                         ("d_raw_opacity", "g_opacity"), ("d_sh", "g_sh"), ("d_raw_mask", "g_mask")):
        a, b = getattr(gb, ours), g[theirs]
        err = grad_rel_error(a, b)
        af, bf = a.ravel(), b.ravel()
        den = np.maximum(np.abs(af), np.abs(bf))
        floor = max(1e-6 * den.max(), 1e-12) if den.size else 1
        rel = np.abs(af - bf) / np.maximum(den, floor)
        worst = np.argsort(rel)[-3:][::-1] if rel.size else []
        print(f"  {ours:14s} err={err:.3e} max|ref|={np.abs(bf).max() if bf.size else 0:.3e} "
              + " ".join(f"[{i}: gpu={af[i]:.4e} ref={bf[i]:.4e} |ref|/max={abs(bf[i])/max(np.abs(bf).max(),1e-30):.1e}]" for i in worst))
    if name == "mode_depth":
        # per-convex breakdown of the worst convex
        a, b = gb.d_points, g["g_points"]
        e = np.abs(a - b).max(axis=(1, 2)) / np.maximum(np.abs(b).max(axis=(1, 2)), 1e-30)
        i = int(np.argmax(e))
        print("   worst convex", i, "gpu\n", a[i], "\n ref\n", b[i])
