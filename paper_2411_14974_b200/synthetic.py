"""Seeded synthetic scenes and cameras (vectorised, SoA).

The benchmark generator G(N, seed) of SURVEY.md section 8(d), following the
reference's conventions (synth.py:60-88 make_scene, initialize.py:33-54
fibonacci_sphere / neighbor_radii): centres uniform in [-1,1]^3 * (1,0.6,1),
radius 1.2x the mean 3-NN distance, six Fibonacci-sphere points + 8% noise,
DC colour in [-1.4,1.4], first SH band N(0, 0.05), delta in [0.8,1.5],
sigma in [0.05,0.12], opacity in [0.75,0.95], mask 0.995.
"""
from __future__ import annotations

import math

import numpy as np

from .model import Camera, inverse_mask_activation, inverse_opacity_activation


def look_at(eye, target=(0.0, 0.0, 0.0), up=(0.0, 1.0, 0.0)):
    """World-to-camera (R, t) with the camera z axis toward ``target``
    (synth.py:19-33 convention: rows right, down, forward)."""
    eye = np.asarray(eye, dtype=np.float64)
    fwd = np.asarray(target, dtype=np.float64) - eye
    fwd /= np.linalg.norm(fwd)
    right = np.cross(np.asarray(up, dtype=np.float64), fwd)
    if np.linalg.norm(right) < 1e-9:
        right = np.cross(np.array([1.0, 0.0, 0.0]), fwd)
    right /= np.linalg.norm(right)
    down = np.cross(fwd, right)
    R = np.stack([right, down, fwd])
    return R, -R @ eye


def bench_camera(width: int, height: int, eye=(0.0, 1.4, -4.0), fov_degrees: float = 50.0) -> Camera:
    """C(W, H) of SURVEY.md 8(d): fx = fy = W / (2 tan(fov/2)), centred."""
    R, t = look_at(eye)
    f = width / (2.0 * math.tan(math.radians(fov_degrees) / 2.0))
    return Camera(fx=f, fy=f, cx=width / 2.0, cy=height / 2.0, width=width, height=height, R=R, t=t)


def ring_cameras(count: int, width: int, height: int = None, radius: float = 4.0, fov_degrees: float = 50.0,
                 elevations=(0.35, -0.2)) -> list:
    """Cameras on a circle, alternating elevation (synth.py:36-57 geometry,
    generalised to W != H)."""
    height = width if height is None else height
    f = width / (2.0 * math.tan(math.radians(fov_degrees) / 2.0))
    cams = []
    for i in range(count):
        a = 2.0 * math.pi * i / count
        el = elevations[i % len(elevations)]
        eye = radius * np.array([math.cos(a) * math.cos(el), math.sin(el), math.sin(a) * math.cos(el)])
        R, t = look_at(eye)
        cams.append(Camera(fx=f, fy=f, cx=width / 2.0, cy=height / 2.0, width=width, height=height, R=R, t=t,
                           image_name=f"view_{i:03d}.png"))
    return cams


def fibonacci_offsets(count: int) -> np.ndarray:
    """Unit Fibonacci-sphere directions (initialize.py:33-42)."""
    golden = math.pi * (3.0 - math.sqrt(5.0))
    i = np.arange(count, dtype=np.float64)
    z = 1.0 - 2.0 * (i + 0.5) / count
    ring = np.sqrt(np.maximum(1.0 - z * z, 0.0))
    th = golden * i
    return np.stack([ring * np.cos(th), ring * np.sin(th), z], axis=1)


def mean_knn_distance(points: np.ndarray, k: int = 3) -> np.ndarray:
    from scipy.spatial import cKDTree
    n = points.shape[0]
    kk = min(k, n - 1)
    if kk <= 0:
        return np.ones(n)
    d, _ = cKDTree(points).query(points, k=kk + 1)
    return d[:, 1:].mean(axis=1)


def generate_scene(n: int, seed: int = 0, k: int = 6) -> dict:
    """G(N, seed) as float64 SoA arrays (quantise to float32 for the GPU)."""
    rng = np.random.default_rng(seed)
    centers = rng.uniform(-1.0, 1.0, size=(n, 3)) * np.array([1.0, 0.6, 1.0])
    radius = 1.2 * mean_knn_distance(centers)
    pts = centers[:, None, :] + radius[:, None, None] * fibonacci_offsets(k)[None]
    pts += rng.normal(0.0, 1.0, size=pts.shape) * (0.08 * radius)[:, None, None]
    sh = np.zeros((n, 16, 3))
    sh[:, 0] = rng.uniform(-1.4, 1.4, size=(n, 3))
    sh[:, 1:4] = rng.normal(0.0, 0.05, size=(n, 3, 3))
    return dict(points=pts, raw_delta=np.log(rng.uniform(0.8, 1.5, size=n)),
                raw_sigma=np.log(rng.uniform(0.05, 0.12, size=n)),
                raw_opacity=inverse_opacity_activation(rng.uniform(0.75, 0.95, size=n)),
                raw_mask=np.full(n, float(inverse_mask_activation(0.995))), sh=sh,
                background=np.zeros(3))


def quantize32(arrays: dict) -> dict:
    """Round every parameter to float32 (so GPU and float64 oracle agree on inputs)."""
    out = {}
    for key, v in arrays.items():
        v = np.asarray(v)
        out[key] = v.astype(np.float32).astype(np.float64) if key != "background" else v
    return out


def perturb(arrays: dict, seed: int = 1, extent: float = 2.0, fraction: float = 0.05) -> dict:
    """Shifted / re-coloured copy used for training targets (synth.py:97-116 idea)."""
    rng = np.random.default_rng(seed)
    n = arrays["points"].shape[0]
    out = {key: np.array(v, copy=True) for key, v in arrays.items()}
    d = rng.normal(size=(n, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    out["points"] += fraction * extent * d[:, None, :]
    out["points"] += rng.normal(0.0, 0.01 * extent, size=out["points"].shape)
    out["sh"][:] = 0.0
    out["sh"][:, 0] = rng.uniform(-1.0, 1.0, size=(n, 3))
    out["raw_opacity"] = inverse_opacity_activation(rng.uniform(0.4, 0.9, size=n))
    out["raw_delta"] = out["raw_delta"] + np.log(rng.uniform(0.8, 1.25, size=n))
    out["raw_sigma"] = out["raw_sigma"] + np.log(rng.uniform(0.8, 1.25, size=n))
    return out


def camera_dict(cam: Camera) -> dict:
    return dict(fx=cam.fx, fy=cam.fy, cx=cam.cx, cy=cam.cy, R=cam.R, t=cam.t, z_near=cam.z_near,
                width=cam.width, height=cam.height, ortho=cam.ortho)
