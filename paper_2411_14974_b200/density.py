"""Adaptive density control on the device:
density.densify_and_prune (density.py:54-105) with split_convex
(density.py:19-43) over the SoA tensors.

Two kernels and two scans: ``cs_density_flags`` decides per convex (float64,
the reference's arithmetic) whether it splits, whether it survives pruning
and which of its K children survive; exclusive scans of the row counts give
every new row its position; ``cs_density_scatter`` writes the new scene in
the reference order (kept survivors in index order, then the kept children of
each split parent in parent order) and the index map Adam.remap needs
(optim.py:37-53).  One host read (the new row count) sizes the outputs.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import torch

from . import _lib
from .rasterizer import params_struct
from .scene_tensors import PARAM_NAMES, SceneTensors


@dataclass
class DensityConfig:
    """The TrainConfig fields densify_and_prune reads (trainer.py:31-39)."""

    densify_stop: int = 9000
    sigma_loss_threshold: float = 4e-6
    prune_opacity: float = 0.03
    prune_size_fraction: float = 0.3
    split_scale: float = 0.7
    split_sigma_boost: float = 1.25
    split_opacity_factor: float = 0.8


@dataclass
class DensifyStats:
    """density.DensifyStats (density.py:46-51)."""

    split: int
    pruned: int
    before: int
    after: int


def densify_and_prune(scene: SceneTensors, sigma_signal: torch.Tensor, config: DensityConfig = DensityConfig(),
                      iteration: int = 0):
    """Returns (new SceneTensors, index_map int64 tensor, DensifyStats); the
    input scene is not modified (the reference edits its list in place)."""
    dev = scene.device
    if dev.type != "cuda":
        raise _lib.CsError("densify_and_prune runs on CUDA devices only (no CPU fallback)")
    n, k = scene.n, scene.k
    signal = sigma_signal.detach().to(device=dev, dtype=torch.float32).contiguous()
    if signal.numel() != n:
        raise ValueError(f"sigma signal has {signal.numel()} entries for {n} convexes")
    cfg = _lib.CsDensityConfig(float(config.sigma_loss_threshold), float(config.split_scale),
                               float(config.split_sigma_boost), float(config.split_opacity_factor),
                               float(config.prune_opacity), float(config.prune_size_fraction * scene.scene_extent),
                               int(iteration <= config.densify_stop), 0)
    p = params_struct(scene)
    flags = torch.empty(n, dtype=torch.uint8, device=dev)
    child_keep = torch.empty(n, dtype=torch.int32, device=dev)
    surv = torch.empty(n, dtype=torch.int64, device=dev)
    kids = torch.empty(n, dtype=torch.int64, device=dev)
    stream = torch.cuda.current_stream(dev).cuda_stream
    L = _lib.load()
    _lib.check(L.cs_density_flags(ctypes.byref(p), signal.data_ptr(), ctypes.byref(cfg), flags.data_ptr(),
                                  child_keep.data_ptr(), surv.data_ptr(), kids.data_ptr(), stream), "cs_density_flags")
    surv_pos = torch.cumsum(surv, 0) - surv          # exclusive scans
    child_pos = torch.cumsum(kids, 0) - kids
    totals = torch.stack([surv.sum(), kids.sum(), (flags >= 2).sum()]).cpu()
    n_surv_kept, n_kids, n_split = (int(v) for v in totals)
    m = n_surv_kept + n_kids
    out = {"points": torch.empty((m, k, 3), device=dev), "sh": torch.empty((m,) + tuple(scene.sh.shape[1:]), device=dev)}
    for f in ("raw_delta", "raw_sigma", "raw_opacity", "raw_mask"):
        out[f] = torch.empty((m,), device=dev)
    index_map = torch.empty(m, dtype=torch.int64, device=dev)
    n_surv_dev = torch.tensor([n_surv_kept], dtype=torch.int64, device=dev)
    so = _lib.CsSceneOut(*(out[f].data_ptr() for f in PARAM_NAMES))
    _lib.check(L.cs_density_scatter(ctypes.byref(p), ctypes.byref(cfg), flags.data_ptr(), child_keep.data_ptr(),
                                    surv_pos.data_ptr(), child_pos.data_ptr(), n_surv_dev.data_ptr(), ctypes.byref(so),
                                    index_map.data_ptr(), stream), "cs_density_scatter")
    new = SceneTensors(**out, background=scene.background.copy(), scene_extent=scene.scene_extent)
    merged = (n - n_split) + n_split * k
    return new, index_map, DensifyStats(split=n_split, pruned=merged - m, before=n, after=m)


__all__ = ["DensityConfig", "DensifyStats", "densify_and_prune"]
