"""Training-step kernels around the rasterizer, bound
through the C ABI (include/convexsplat_b200.h):

* ``image_loss``   losses.image_loss (losses.py:129-155): fused L1 + D-SSIM
  (11x11 Gaussian, valid window) value and d_image, mask term and its
  gradient, in three kernels (cs_image_loss); the scalars stay on the device.
* ``FusedAdam``    optim.Adam (optim.py:12-53): one launch updates every
  parameter tensor (cs_adam_step); ``remap`` follows densification rows.

CUDA only, like the renderer: there is no CPU path here (the torch
formulations in ``sharded`` are the reference the tests compare against).
"""
from __future__ import annotations

import ctypes
from typing import Optional

import torch

from . import _lib

PARAM_ORDER = ("points", "raw_delta", "raw_sigma", "raw_opacity", "sh", "raw_mask")


def _cuda_f32(t: torch.Tensor, name: str) -> torch.Tensor:
    if t.device.type != "cuda" or t.dtype != torch.float32 or not t.is_contiguous():
        raise ValueError(f"{name} must be a contiguous float32 CUDA tensor")
    return t


class LossWorkspace:
    """Scratch of cs_image_loss (9 coefficient maps of the valid SSIM grid)."""

    def __init__(self):
        self.buffer: Optional[torch.Tensor] = None
        self.stats: Optional[torch.Tensor] = None

    def ensure(self, height: int, width: int, device) -> None:
        nbytes = ctypes.c_size_t()
        _lib.check(_lib.load().cs_image_loss_workspace(height, width, ctypes.byref(nbytes)), "cs_image_loss_workspace")
        if self.buffer is None or self.buffer.numel() < nbytes.value or self.buffer.device != torch.device(device):
            self.buffer = torch.empty(max(nbytes.value, 16), dtype=torch.uint8, device=device)
        if self.stats is None or self.stats.device != torch.device(device):
            self.stats = torch.zeros(9, dtype=torch.float64, device=device)


def image_loss(rendered: torch.Tensor, target: torch.Tensor, raw_mask: torch.Tensor, lambda_dssim: float = 0.2,
               beta_mask: float = 0.0005, d_raw_mask: Optional[torch.Tensor] = None,
               workspace: Optional[LossWorkspace] = None) -> dict:
    """(1 - lambda) L1 + lambda (1 - SSIM)/2 + beta mean(sigmoid(raw_mask))
    (losses.py:129-155) on (H, W, 3) images.  Returns device scalars
    (total, l1, dssim, mask_term) and d_image; the mask gradient
    beta m (1-m) / n is ADDED to ``d_raw_mask`` when given (trainer.py:176)."""
    if rendered.shape != target.shape or rendered.dim() != 3 or rendered.shape[2] != 3:
        raise ValueError(f"shape mismatch {tuple(rendered.shape)} vs {tuple(target.shape)}")
    H, W = int(rendered.shape[0]), int(rendered.shape[1])
    if H < 11 or W < 11:
        raise ValueError("image smaller than the 11x11 SSIM window")   # losses.py:60-63
    _cuda_f32(rendered, "rendered")
    _cuda_f32(target, "target")
    _cuda_f32(raw_mask, "raw_mask")
    if d_raw_mask is not None:
        _cuda_f32(d_raw_mask, "d_raw_mask")
    ws = workspace or LossWorkspace()
    ws.ensure(H, W, rendered.device)
    d_image = torch.empty_like(rendered)
    stream = torch.cuda.current_stream(rendered.device).cuda_stream
    n = int(raw_mask.numel())
    _lib.check(_lib.load().cs_image_loss(H, W, rendered.data_ptr(), target.data_ptr(),
                                         raw_mask.data_ptr() if n else None, n, float(lambda_dssim),
                                         float(beta_mask), d_image.data_ptr(),
                                         d_raw_mask.data_ptr() if d_raw_mask is not None else None,
                                         ws.stats.data_ptr(), ws.buffer.data_ptr(), ws.buffer.numel(), stream),
               "cs_image_loss")
    st = ws.stats.clone()   # values formed on the device (stats[4:9]); the clone survives the next call
    return {"total": st[4], "l1": st[5], "dssim": st[7], "ssim": st[6], "mask_term": st[8], "d_image": d_image}


class FusedAdam:
    """optim.Adam (optim.py:12-53) over the named parameter tensors, one
    cs_adam_step launch per step."""

    def __init__(self, params: dict, beta1: float = 0.9, beta2: float = 0.999, eps: float = 1e-15):
        self.beta1, self.beta2, self.eps = beta1, beta2, eps
        self.step_count = 0
        for k, v in params.items():
            _cuda_f32(v, k)
        self.m = {k: torch.zeros_like(v) for k, v in params.items()}
        self.v = {k: torch.zeros_like(v) for k, v in params.items()}

    @torch.no_grad()
    def step(self, params: dict, grads: dict, lrs: dict, grad_scale: float = 1.0):
        """In place on ``params``; the gradient is multiplied by grad_scale
        first (1/B of the view-sharded step)."""
        self.step_count += 1
        names = list(params)
        arr = (_lib.CsAdamTensor * len(names))()
        for j, name in enumerate(names):
            p, g = params[name], _cuda_f32(grads[name], f"grad {name}")
            if g.shape != p.shape:
                raise ValueError(f"gradient {name} has shape {tuple(g.shape)}, parameter {tuple(p.shape)}")
            arr[j] = _lib.CsAdamTensor(p.data_ptr(), g.data_ptr(), self.m[name].data_ptr(), self.v[name].data_ptr(),
                                       p.numel(), float(lrs[name]))
        stream = torch.cuda.current_stream(params[names[0]].device).cuda_stream
        _lib.check(_lib.load().cs_adam_step(len(names), arr, self.beta1, self.beta2, self.eps, self.step_count,
                                            float(grad_scale), stream), "cs_adam_step")

    @torch.no_grad()
    def remap(self, index_map: torch.Tensor):
        """optim.py:37-53: new row j takes old row index_map[j]; -1 = fresh zeros."""
        index_map = index_map.to(device=next(iter(self.m.values())).device, dtype=torch.int64)
        keep = index_map >= 0
        for name in self.m:
            for store in (self.m, self.v):
                old = store[name]
                new = torch.zeros((index_map.numel(),) + tuple(old.shape[1:]), dtype=old.dtype, device=old.device)
                new[keep] = old[index_map[keep]]
                store[name] = new


__all__ = ["image_loss", "LossWorkspace", "FusedAdam", "PARAM_ORDER"]
