"""Scene, camera and settings types of the drop-in API.

Same names, fields, defaults and validation errors as the reference package
(model.py:57-194, rasterize.py:23-74, field.py:17-23, backward.py:39-73) so
reference callers keep working; internally the renderer consumes the
structure-of-arrays ``SceneTensors`` (float32, on the GPU), which is the
primary representation for large scenes.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from enum import Enum
from typing import Optional

import numpy as np

SH_COEFFS = 16          # model.py:15  (degree-3 real SH, per colour channel)
MIN_POINTS = 4          # model.py:18
TILE_SIZE = 16          # rasterize.py:23
MASK_GATE = 0.01        # rasterize.py:26
ALPHA_MAX = 1.0 - 1e-6  # rasterize.py:30


def _sigmoid(x):
    return 1.0 / (1.0 + np.exp(-np.asarray(x, dtype=np.float64)))


def _logit(p):
    p = np.asarray(p, dtype=np.float64)
    return np.log(p) - np.log1p(-p)


# Activations and inverses (model.py:21-54).
def delta_activation(raw):
    return np.exp(raw)


def sigma_activation(raw):
    return np.exp(raw)


def opacity_activation(raw):
    return _sigmoid(raw)


def mask_activation(raw):
    return _sigmoid(raw)


def inverse_delta_activation(value):
    return np.log(value)


def inverse_sigma_activation(value):
    return np.log(value)


def inverse_opacity_activation(value):
    return _logit(value)


def inverse_mask_activation(value):
    return _logit(value)


class ScalingMode(Enum):
    """Depth multiplier of delta and sigma (field.py:17-23)."""

    NONE = "none"
    SQRT_DEPTH = "sqrt"
    DEPTH = "depth"
    DEPTH_SQUARED = "depth2"

    @property
    def code(self) -> int:  # enum cs_scaling of include/convexsplat_b200.h
        return {"none": 0, "sqrt": 1, "depth": 2, "depth2": 3}[self.value]

    @classmethod
    def of(cls, mode) -> "ScalingMode":
        """This enum from itself, its value string, or any enum with the same
        values (the reference's field.ScalingMode: drop-in callers pass it)."""
        return cls(getattr(mode, "value", mode))


@dataclass(frozen=True)
class RenderSettings:
    """rasterize.py:33-50.  tile_size 16 is the value the sm_100a kernels support."""

    contribution_cutoff: float = 2e-4
    transmittance_floor: float = 1e-4
    tile_size: int = TILE_SIZE
    sh_degree: int = 3


EXACT_SETTINGS = RenderSettings(contribution_cutoff=0.0, transmittance_floor=0.0)  # rasterize.py:53


@dataclass
class SmoothConvex:
    """K points + raw appearance parameters (model.py:57-126)."""

    points: np.ndarray
    raw_delta: float
    raw_sigma: float
    raw_opacity: float
    sh: np.ndarray
    raw_mask: float

    def __post_init__(self):
        self.points = np.asarray(self.points, dtype=np.float64)
        if self.points.ndim != 2 or self.points.shape[1] != 3:
            raise ValueError(f"points must be (K, 3), got {self.points.shape}")
        if self.points.shape[0] < MIN_POINTS:
            raise ValueError(f"a smooth convex needs at least {MIN_POINTS} points, "
                             f"got {self.points.shape[0]}")
        self.sh = np.asarray(self.sh, dtype=np.float64)
        if self.sh.shape != (SH_COEFFS, 3):
            raise ValueError(f"sh must be ({SH_COEFFS}, 3), got {self.sh.shape}")

    @property
    def num_points(self) -> int:
        return self.points.shape[0]

    @property
    def delta(self) -> float:
        return float(np.exp(self.raw_delta))

    @property
    def sigma(self) -> float:
        return float(np.exp(self.raw_sigma))

    @property
    def opacity(self) -> float:
        return float(_sigmoid(self.raw_opacity))

    @property
    def mask(self) -> float:
        return float(_sigmoid(self.raw_mask))

    def center(self) -> np.ndarray:
        return self.points.mean(axis=0)

    def diameter(self) -> float:
        d = self.points[:, None, :] - self.points[None, :, :]
        return float(np.sqrt((d * d).sum(axis=2)).max())

    def copy(self) -> "SmoothConvex":
        return SmoothConvex(self.points.copy(), float(self.raw_delta), float(self.raw_sigma),
                            float(self.raw_opacity), self.sh.copy(), float(self.raw_mask))


@dataclass
class Camera:
    """Pinhole/orthographic camera, x_cam = R p + t (model.py:135-172)."""

    fx: float
    fy: float
    cx: float
    cy: float
    width: int
    height: int
    R: np.ndarray
    t: np.ndarray
    z_near: float = 0.01
    ortho: bool = False
    image_name: str = ""

    def __post_init__(self):
        self.R = np.asarray(self.R, dtype=np.float64).reshape(3, 3)
        self.t = np.asarray(self.t, dtype=np.float64).reshape(3)

    def world_to_cam(self, points: np.ndarray) -> np.ndarray:
        return np.asarray(points, dtype=np.float64) @ self.R.T + self.t

    def center(self) -> np.ndarray:
        return -self.R.T @ self.t

    def pixel_grid(self):
        return (np.arange(self.width, dtype=np.float64) + 0.5,
                np.arange(self.height, dtype=np.float64) + 0.5)


@dataclass
class Scene:
    """Primitive list + background (model.py:175-194)."""

    primitives: list
    background: np.ndarray = field(default_factory=lambda: np.zeros(3))
    scene_extent: float = 1.0

    def __post_init__(self):
        self.background = np.asarray(self.background, dtype=np.float64).reshape(3)

    def __len__(self) -> int:
        return len(self.primitives)

    def copy(self) -> "Scene":
        return Scene([p.copy() for p in self.primitives], self.background.copy(),
                     float(self.scene_extent))


@dataclass
class RenderOutput:
    """rasterize.py:68-74, plus ``depth`` (sum over blends of T*alpha*depth)."""

    image: np.ndarray
    final_transmittance: np.ndarray
    per_pixel_count: np.ndarray
    blend_weight_sum: np.ndarray
    visible: np.ndarray = None
    depth: Optional[np.ndarray] = None


@dataclass
class GradientBuffer:
    """Per-primitive gradients w.r.t. raw parameters (backward.py:39-73)."""

    d_points: np.ndarray
    d_raw_delta: np.ndarray
    d_raw_sigma: np.ndarray
    d_raw_opacity: np.ndarray
    d_sh: np.ndarray
    d_raw_mask: np.ndarray
    visible: np.ndarray

    @classmethod
    def zeros(cls, scene) -> "GradientBuffer":
        n = len(scene)
        k = _num_points(scene)
        return cls(np.zeros((n, k, 3)), np.zeros(n), np.zeros(n), np.zeros(n),
                   np.zeros((n, SH_COEFFS, 3)), np.zeros(n), np.zeros(n, dtype=bool))

    def add(self, other: "GradientBuffer") -> "GradientBuffer":
        for name in ("d_points", "d_raw_delta", "d_raw_sigma", "d_raw_opacity", "d_sh", "d_raw_mask"):
            getattr(self, name).__iadd__(getattr(other, name))
        self.visible |= other.visible
        return self


def _num_points(scene) -> int:
    if hasattr(scene, "points") and not isinstance(scene, Scene):
        return int(scene.points.shape[1])
    return scene.primitives[0].num_points if len(scene.primitives) else 0
