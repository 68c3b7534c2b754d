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


# ----------------------------------------------------------------------------- config 2: toy chair
# BASELINE.json configs[1] / SURVEY.md 8(d) row 2.  The paper's chair
# (Fig. 2) is a 2-D toy; this is a procedural 3-D chair -- a seat, a back
# and four legs -- whose parts are boxes split into 6-point triangular
# prisms (two per box cell), the ground truth the fit is rendered from.
SH_C0 = 0.28209479177387814   # harmonics.py:7 (degree-0 SH constant)
CHAIR_PARTS = (
    # (min corner, max corner, colour, cells per axis)
    ((-0.6, -0.05, -0.6), (0.6, 0.1, 0.6), (0.75, 0.45, 0.2), (4, 1, 4)),      # seat
    ((-0.6, 0.1, 0.45), (0.6, 1.2, 0.6), (0.55, 0.3, 0.15), (4, 4, 1)),        # back
    ((-0.55, -1.0, -0.55), (-0.4, -0.05, -0.4), (0.3, 0.3, 0.35), (1, 3, 1)),  # legs
    ((0.4, -1.0, -0.55), (0.55, -0.05, -0.4), (0.3, 0.3, 0.35), (1, 3, 1)),
    ((-0.55, -1.0, 0.4), (-0.4, -0.05, 0.55), (0.3, 0.3, 0.35), (1, 3, 1)),
    ((0.4, -1.0, 0.4), (0.55, -0.05, 0.55), (0.3, 0.3, 0.35), (1, 3, 1)),
)


def _prisms_of_box(lo, hi) -> list:
    """A box as two triangular prisms (6 points each): the x-z rectangle split
    along its diagonal, extruded along y."""
    (x0, y0, z0), (x1, y1, z1) = lo, hi
    tris = (((x0, z0), (x1, z0), (x1, z1)), ((x0, z0), (x1, z1), (x0, z1)))
    return [np.array([(x, y0, z) for x, z in t] + [(x, y1, z) for x, z in t], dtype=np.float64) for t in tris]


def chair_scene(opacity: float = 0.98, delta: float = 20.0, sigma: float = 0.05) -> dict:
    """Ground-truth chair as SoA arrays (sharp, nearly opaque prisms)."""
    pts, cols = [], []
    for lo, hi, col, cells in CHAIR_PARTS:
        lo, hi = np.asarray(lo), np.asarray(hi)
        step = (hi - lo) / np.asarray(cells)
        for ix in range(cells[0]):
            for iy in range(cells[1]):
                for iz in range(cells[2]):
                    a = lo + step * (ix, iy, iz)
                    for prism in _prisms_of_box(a, a + step):
                        pts.append(prism)
                        cols.append(col)
    n = len(pts)
    sh = np.zeros((n, 16, 3))
    sh[:, 0] = (np.asarray(cols) - 0.5) / SH_C0
    return dict(points=np.stack(pts), raw_delta=np.full(n, math.log(delta)), raw_sigma=np.full(n, math.log(sigma)),
                raw_opacity=np.full(n, float(inverse_opacity_activation(opacity))),
                raw_mask=np.full(n, float(inverse_mask_activation(0.995))), sh=sh, background=np.zeros(3))


def chair_surface_samples(count: int = 2000, seed: int = 0, noise: float = 0.02):
    """~count points on the chair's box surfaces (area-weighted) with their
    part colours (+ noise): the sparse point cloud of initialize.init_scene."""
    rng = np.random.default_rng(seed)
    faces = []
    for lo, hi, col, _ in CHAIR_PARTS:
        lo, hi = np.asarray(lo, dtype=np.float64), np.asarray(hi, dtype=np.float64)
        for axis in range(3):
            u, v = [a for a in range(3) if a != axis]
            area = (hi[u] - lo[u]) * (hi[v] - lo[v])
            for side in (lo[axis], hi[axis]):
                faces.append((axis, side, lo, hi, u, v, area, col))
    areas = np.array([f[6] for f in faces])
    pick = rng.choice(len(faces), size=count, p=areas / areas.sum())
    pts = np.empty((count, 3))
    cols = np.empty((count, 3))
    for j, fi in enumerate(pick):
        axis, side, lo, hi, u, v, _, col = faces[fi]
        pts[j, axis] = side
        pts[j, u] = rng.uniform(lo[u], hi[u])
        pts[j, v] = rng.uniform(lo[v], hi[v])
        cols[j] = col
    cols = np.clip(cols + rng.normal(0.0, noise, size=cols.shape), 0.0, 1.0)
    return pts, cols


def init_scene_arrays(points: np.ndarray, colors: np.ndarray, k: int = 6) -> dict:
    """initialize.init_scene (initialize.py:67-106) as SoA arrays: one convex
    per point on a Fibonacci sphere of radius 1.2 x the mean 3-NN distance,
    delta 0.1, sigma 0.00095, opacity 0.1, mask 0.99, SH DC from the colour."""
    from .model import inverse_delta_activation, inverse_sigma_activation
    points = np.asarray(points, dtype=np.float64).reshape(-1, 3)
    n = points.shape[0]
    radii = np.maximum(1.2 * mean_knn_distance(points), 1e-9)
    pts = points[:, None, :] + radii[:, None, None] * fibonacci_offsets(k)[None]
    sh = np.zeros((n, 16, 3))
    sh[:, 0] = (np.asarray(colors, dtype=np.float64) - 0.5) / SH_C0
    return dict(points=pts, raw_delta=np.full(n, float(inverse_delta_activation(0.1))),
                raw_sigma=np.full(n, float(inverse_sigma_activation(0.00095))),
                raw_opacity=np.full(n, float(inverse_opacity_activation(0.1))),
                raw_mask=np.full(n, float(inverse_mask_activation(0.99))), sh=sh, background=np.zeros(3))
