"""Structure-of-arrays scene on the GPU (the renderer's native input).

A list of 1M ``SmoothConvex`` objects costs ~1 min to build in Python; large
scenes therefore live as float32 SoA tensors:

    points [N,K,3], raw_delta/raw_sigma/raw_opacity/raw_mask [N], sh [N,16,3]

``from_scene``/``to_scene`` convert to and from the reference-compatible
``Scene`` (model.py:175-194).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np
import torch

from .model import SH_COEFFS, Scene, SmoothConvex

PARAM_NAMES = ("points", "raw_delta", "raw_sigma", "raw_opacity", "raw_mask", "sh")


@dataclass
class SceneTensors:
    points: torch.Tensor
    raw_delta: torch.Tensor
    raw_sigma: torch.Tensor
    raw_opacity: torch.Tensor
    raw_mask: torch.Tensor
    sh: torch.Tensor
    background: np.ndarray = None
    scene_extent: float = 1.0

    def __post_init__(self):
        if self.background is None:
            self.background = np.zeros(3)
        self.background = np.asarray(self.background, dtype=np.float64).reshape(3)
        n = self.points.shape[0]
        if self.points.dim() != 3 or self.points.shape[2] != 3:
            raise ValueError(f"points must be (N, K, 3), got {tuple(self.points.shape)}")
        if tuple(self.sh.shape) != (n, SH_COEFFS, 3):
            raise ValueError(f"sh must be (N, {SH_COEFFS}, 3), got {tuple(self.sh.shape)}")
        for name in ("raw_delta", "raw_sigma", "raw_opacity", "raw_mask"):
            if tuple(getattr(self, name).shape) != (n,):
                raise ValueError(f"{name} must be ({n},)")

    def __len__(self) -> int:
        return int(self.points.shape[0])

    @property
    def n(self) -> int:
        return int(self.points.shape[0])

    @property
    def k(self) -> int:
        return int(self.points.shape[1])

    @property
    def device(self) -> torch.device:
        return self.points.device

    def params(self) -> tuple:
        return tuple(getattr(self, f) for f in PARAM_NAMES)

    def to(self, device, dtype=torch.float32) -> "SceneTensors":
        kw = {f: getattr(self, f).to(device=device, dtype=dtype).contiguous() for f in PARAM_NAMES}
        return SceneTensors(**kw, background=self.background.copy(), scene_extent=self.scene_extent)

    def detach(self) -> "SceneTensors":
        kw = {f: getattr(self, f).detach() for f in PARAM_NAMES}
        return SceneTensors(**kw, background=self.background.copy(), scene_extent=self.scene_extent)

    def numpy(self) -> dict:
        return {f: getattr(self, f).detach().double().cpu().numpy() for f in PARAM_NAMES}

    @classmethod
    def from_arrays(cls, arrays: dict, device="cuda", background=None, scene_extent=1.0) -> "SceneTensors":
        kw = {f: torch.as_tensor(np.asarray(arrays[f]), dtype=torch.float32).to(device).contiguous()
              for f in PARAM_NAMES}
        return cls(**kw, background=background if background is not None else arrays.get("background"),
                   scene_extent=scene_extent)

    @classmethod
    def from_scene(cls, scene: Scene, device="cuda") -> "SceneTensors":
        prims = list(scene.primitives)
        k = int(np.asarray(prims[0].points).shape[0]) if prims else 6
        arrays = dict(
            points=np.stack([c.points for c in prims]) if prims else np.zeros((0, k, 3)),
            raw_delta=np.array([c.raw_delta for c in prims], dtype=np.float64),
            raw_sigma=np.array([c.raw_sigma for c in prims], dtype=np.float64),
            raw_opacity=np.array([c.raw_opacity for c in prims], dtype=np.float64),
            raw_mask=np.array([c.raw_mask for c in prims], dtype=np.float64),
            sh=np.stack([c.sh for c in prims]) if prims else np.zeros((0, SH_COEFFS, 3)),
        )
        return cls.from_arrays(arrays, device, np.asarray(getattr(scene, "background", np.zeros(3)), dtype=np.float64),
                               float(getattr(scene, "scene_extent", 1.0)))

    def to_scene(self) -> Scene:
        a = self.numpy()
        prims = [SmoothConvex(a["points"][i], float(a["raw_delta"][i]), float(a["raw_sigma"][i]),
                              float(a["raw_opacity"][i]), a["sh"][i], float(a["raw_mask"][i]))
                 for i in range(self.n)]
        return Scene(prims, self.background.copy(), self.scene_extent)


def as_scene_tensors(scene, device: Optional[torch.device] = None) -> SceneTensors:
    """Accept a Scene or SceneTensors; returns float32 SceneTensors on ``device``."""
    device = device or torch.device("cuda")
    if isinstance(scene, SceneTensors):
        if scene.device != device or scene.points.dtype != torch.float32:
            return scene.to(device)
        return scene
    if isinstance(scene, Scene) or hasattr(scene, "primitives"):
        # this package's Scene, or any object with the reference Scene's
        # surface (model.py:175-194: primitives of SmoothConvex-like objects
        # with points / raw_* / sh, background, scene_extent) -- the
        # reference's own convexsplat.model.Scene is accepted as is
        return SceneTensors.from_scene(scene, device)
    raise TypeError(f"expected a Scene (with .primitives) or SceneTensors, got {type(scene).__name__}")


__all__ = ["SceneTensors", "PARAM_NAMES", "as_scene_tensors"]
