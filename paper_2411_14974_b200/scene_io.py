""".3dcs checkpoints straight into / out of the SoA device tensors (SURVEY
8(f) row 4; sceneio.py:251-320).

The reference builds one ``SmoothConvex`` per row (about a minute for a 1M
scene); here the host only parses the 64-byte header and moves the raw
payload, and ``cs_checkpoint_unpack`` / ``cs_checkpoint_pack`` convert rows
<-> SoA on the device (float16 rows are rounded to nearest even, like
numpy's ``astype('<f2')``).  File format, validation order and error types
follow the reference: header ``<4sIIIII4d`` = magic "3DCS", version 1,
precision 16|32, count, K, SH degree 3, background[3], scene extent.
"""
from __future__ import annotations

import ctypes
import struct
from pathlib import Path

import numpy as np
import torch

from . import _lib
from .model import SH_COEFFS
from .scene_tensors import PARAM_NAMES, SceneTensors

CHECKPOINT_MAGIC = b"3DCS"
CHECKPOINT_VERSION = 1
_HEADER = struct.Struct("<4sIIIII4d")   # sceneio.py:23


class CheckpointFormatError(ValueError):
    """sceneio.CheckpointFormatError (sceneio.py:33-34)."""


def _params_per_primitive(num_points: int) -> int:
    return 3 * num_points + 3 + 3 * SH_COEFFS + 1   # sceneio.py:251-252


def _scene_out(arrays: dict) -> _lib.CsSceneOut:
    return _lib.CsSceneOut(*(arrays[f].data_ptr() for f in PARAM_NAMES))


def read_header(raw: bytes, path="<bytes>") -> dict:
    """Validate like sceneio.load_checkpoint (sceneio.py:282-301)."""
    if len(raw) < _HEADER.size:
        raise CheckpointFormatError(f"{path}: file too small for header")
    magic, version, precision, count, num_points, _sh, b0, b1, b2, extent = _HEADER.unpack_from(raw)
    if magic != CHECKPOINT_MAGIC:
        raise CheckpointFormatError(f"{path}: bad magic {magic!r}")
    if version != CHECKPOINT_VERSION:
        raise CheckpointFormatError(f"{path}: unsupported version {version} (expected {CHECKPOINT_VERSION})")
    if precision not in (16, 32):
        raise CheckpointFormatError(f"{path}: bad precision {precision}")
    per = _params_per_primitive(num_points)
    itemsize = 4 if precision == 32 else 2
    expected = _HEADER.size + count * per * itemsize
    if len(raw) != expected:
        raise CheckpointFormatError(f"{path}: payload is {len(raw)} bytes, expected {expected}")
    return dict(precision=precision, count=count, k=num_points, background=np.array([b0, b1, b2]),
                scene_extent=float(extent), itemsize=itemsize)


def load_checkpoint(path, device="cuda") -> SceneTensors:
    """sceneio.load_checkpoint -> SoA float32 tensors on ``device`` (CUDA)."""
    raw = Path(path).read_bytes()
    h = read_header(raw, path)
    n, k = h["count"], h["k"]
    if not 3 <= k <= 16:
        raise CheckpointFormatError(f"{path}: {k} points per convex is outside 3..16")
    dev = torch.device(device)
    if dev.type != "cuda":
        raise _lib.CsError("checkpoint unpacking runs on CUDA devices only (no CPU fallback)")
    arrays = {"points": torch.empty((n, k, 3), device=dev), "sh": torch.empty((n, SH_COEFFS, 3), device=dev)}
    for f in ("raw_delta", "raw_sigma", "raw_opacity", "raw_mask"):
        arrays[f] = torch.empty((n,), device=dev)
    if n:
        host = torch.frombuffer(bytearray(raw[_HEADER.size:]), dtype=torch.uint8)
        rows = host.pin_memory().to(dev, non_blocking=True)
        stream = torch.cuda.current_stream(dev).cuda_stream
        _lib.check(_lib.load().cs_checkpoint_unpack(h["precision"], n, k, rows.data_ptr(),
                                                    ctypes.byref(_scene_out(arrays)), stream), "cs_checkpoint_unpack")
        torch.cuda.current_stream(dev).synchronize()
    return SceneTensors(**arrays, background=h["background"], scene_extent=h["scene_extent"])


def save_checkpoint(path, scene: SceneTensors, precision: int = 32) -> None:
    """sceneio.save_checkpoint (sceneio.py:255-279) from SoA tensors: byte-
    identical to the reference for the same (float32) parameter values."""
    if precision not in (16, 32):
        raise ValueError(f"precision must be 16 or 32, got {precision}")
    if scene.n == 0:
        raise ValueError("refusing to save an empty scene")
    dev = scene.device
    if dev.type != "cuda":
        raise _lib.CsError("checkpoint packing runs on CUDA devices only (no CPU fallback)")
    n, k = scene.n, scene.k
    arrays = {f: getattr(scene, f).detach().to(torch.float32).contiguous() for f in PARAM_NAMES}
    itemsize = 4 if precision == 32 else 2
    rows = torch.empty(n * _params_per_primitive(k) * itemsize, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev).cuda_stream
    _lib.check(_lib.load().cs_checkpoint_pack(precision, n, k, ctypes.byref(_scene_out(arrays)), rows.data_ptr(),
                                              stream), "cs_checkpoint_pack")
    payload = rows.cpu().numpy().tobytes()
    bg = np.asarray(scene.background, dtype=np.float64)
    header = _HEADER.pack(CHECKPOINT_MAGIC, CHECKPOINT_VERSION, precision, n, k, 3, float(bg[0]), float(bg[1]),
                          float(bg[2]), float(scene.scene_extent))
    with open(path, "wb") as f:
        f.write(header)
        f.write(payload)


__all__ = ["load_checkpoint", "save_checkpoint", "read_header", "CheckpointFormatError", "CHECKPOINT_MAGIC",
           "CHECKPOINT_VERSION"]
