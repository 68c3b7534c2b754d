"""Loaders for the reference-generated golden fixtures (tests/golden/*.npz)."""
from __future__ import annotations

import glob
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def scene_cases():
    return sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, "*.npz"))
                  if not p.endswith(("hulls.npz", "loss.npz", "ckpt.npz", "density.npz")))


def load(name: str) -> dict:
    with np.load(os.path.join(GOLDEN, f"{name}.npz"), allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


def params(g: dict) -> dict:
    return {k: g[k] for k in ("points", "raw_delta", "raw_sigma", "raw_opacity", "raw_mask", "sh")}


def camera(g: dict) -> dict:
    fx, fy, cx, cy, z_near = (float(v) for v in g["cam_intr"])
    w, h, ortho = (int(v) for v in g["cam_size"])
    return dict(fx=fx, fy=fy, cx=cx, cy=cy, z_near=z_near, R=g["cam_R"], t=g["cam_t"],
                width=w, height=h, ortho=bool(ortho))


def settings(g: dict) -> dict:
    cut, flo = (float(v) for v in g["set_cut_floor"])
    tile, deg = (int(v) for v in g["set_ints"])
    return dict(cutoff=cut, floor=flo, tile=tile, sh_degree=deg, mode=str(g["set_mode"]),
                background=g["background"])
