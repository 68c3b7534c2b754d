"""View-sharded training step (north_star item 5).

One process per GPU.  A batch of B views is split round-robin (view i goes to
rank i mod G).  Each rank renders its views, evaluates the reference training
loss on the device, and accumulates the per-view gradients straight into one
flat float32 buffer (the C ABI accumulates, matching GradientBuffer.add,
backward.py:65-73).  The per-view sigma signal of trainer.py:192-193
(|d_raw_sigma| * visible and the visible-view count) is accumulated beside it,
because it cannot be formed from the summed gradient.  One all_reduce(SUM)
over NCCL combines the buffer; every rank then applies the identical Adam step
(optim.py:12-35, position schedule optim.py:56-61), so replicas stay equal.

On the GPU the loss (losses.py:129-155: L1 + D-SSIM with an 11x11 sigma-1.5
Gaussian valid window + beta * mean sigmoid(mask)) and its image gradient come
from the fused CUDA kernels of ``train_ops`` and the update from one fused
Adam launch; the torch formulation below (``image_loss``, ``Adam``) is the
reference the tests compare against and the CPU (gloo) tests use.
"""
from __future__ import annotations

import math
import os
from dataclasses import dataclass
from typing import Callable, Optional

import torch
import torch.distributed as dist
import torch.nn.functional as F

PARAM_ORDER = ("points", "raw_delta", "raw_sigma", "raw_opacity", "sh", "raw_mask")
GROUP_OF = {"points": "points", "raw_delta": "delta", "raw_sigma": "sigma", "raw_opacity": "opacity",
            "sh": "sh", "raw_mask": "mask"}


@dataclass
class StepConfig:
    """Subset of trainer.TrainConfig (trainer.py:19-62) the step uses."""

    total_iterations: int = 30000
    lambda_dssim: float = 0.2
    beta_mask: float = 0.0005
    lr_position_init: float = 5e-4
    lr_position_final: float = 5e-6
    lr_delta: float = 0.005
    lr_sigma: float = 0.0045
    lr_opacity: float = 0.05
    lr_sh: float = 0.0025
    lr_mask: float = 0.01


# --------------------------------------------------------------------------- loss (losses.py)
SSIM_C1, SSIM_C2 = 0.01 ** 2, 0.03 ** 2


def gaussian_window(size: int = 11, sigma: float = 1.5, device=None, dtype=torch.float32) -> torch.Tensor:
    """losses.py:22-25"""
    off = torch.arange(size, dtype=torch.float64) - (size - 1) / 2.0
    g = torch.exp(-(off ** 2) / (2.0 * sigma * sigma))
    return (g / g.sum()).to(device=device, dtype=dtype)


def _filter_valid(x: torch.Tensor, w: torch.Tensor) -> torch.Tensor:
    """Separable valid-window Gaussian mean (losses.py:31-42); x: [C, H, W]."""
    k = w.numel()
    x = x.unsqueeze(1)
    x = F.conv2d(x, w.view(1, 1, k, 1))
    x = F.conv2d(x, w.view(1, 1, 1, k))
    return x.squeeze(1)


def ssim(img: torch.Tensor, target: torch.Tensor, window: Optional[torch.Tensor] = None) -> torch.Tensor:
    """Mean SSIM of two [H, W, 3] images (losses.py:58-84), differentiable."""
    if img.shape != target.shape:
        raise ValueError(f"shape mismatch {tuple(img.shape)} vs {tuple(target.shape)}")
    if img.shape[0] < 11 or img.shape[1] < 11:
        raise ValueError("image smaller than the 11x11 SSIM window")
    w = window if window is not None else gaussian_window(device=img.device, dtype=img.dtype)
    x, y = img.permute(2, 0, 1), target.permute(2, 0, 1)
    mx, my = _filter_valid(x, w), _filter_valid(y, w)
    sxx = _filter_valid(x * x, w) - mx * mx
    syy = _filter_valid(y * y, w) - my * my
    sxy = _filter_valid(x * y, w) - mx * my
    smap = ((2 * mx * my + SSIM_C1) * (2 * sxy + SSIM_C2)) / ((mx * mx + my * my + SSIM_C1) * (sxx + syy + SSIM_C2))
    return smap.mean(dim=(1, 2)).mean()


def image_loss(img: torch.Tensor, target: torch.Tensor, raw_mask: torch.Tensor, lambda_dssim: float = 0.2,
               beta_mask: float = 0.0005) -> dict:
    """(1-lambda) L1 + lambda (1-SSIM)/2 + beta mean(sigmoid(raw_mask)) (losses.py:129-155)."""
    l1 = (img - target).abs().mean()
    dssim = (1.0 - ssim(img, target)) / 2.0
    mask_term = torch.sigmoid(raw_mask).mean() if raw_mask.numel() else img.new_zeros(())
    total = (1.0 - lambda_dssim) * l1 + lambda_dssim * dssim + beta_mask * mask_term
    return {"total": total, "l1": l1, "dssim": dssim, "mask_term": mask_term}


# --------------------------------------------------------------------------- optimiser (optim.py)
def position_lr(iteration: int, lr_init: float, lr_final: float, total: int) -> float:
    """optim.py:56-61"""
    if total <= 0:
        return lr_init
    frac = min(max(iteration / total, 0.0), 1.0)
    return float(lr_init * (lr_final / lr_init) ** frac)


class Adam:
    """optim.py:12-35 over the parameter tensors, in place, via foreach kernels."""

    def __init__(self, params: dict, beta1: float = 0.9, beta2: float = 0.999, eps: float = 1e-15):
        self.beta1, self.beta2, self.eps = beta1, beta2, eps
        self.step_count = 0
        self.m = {k: torch.zeros_like(v) for k, v in params.items()}
        self.v = {k: torch.zeros_like(v) for k, v in params.items()}

    @torch.no_grad()
    def step(self, params: dict, grads: dict, lrs: dict, grad_scale: float = 1.0):
        self.step_count += 1
        bc1 = 1.0 - self.beta1 ** self.step_count
        bc2 = 1.0 - self.beta2 ** self.step_count
        for name, p in params.items():
            g, m, v = grads[name], self.m[name], self.v[name]
            if grad_scale != 1.0:
                g = g * grad_scale
            m.mul_(self.beta1).add_(g, alpha=1.0 - self.beta1)
            v.mul_(self.beta2).addcmul_(g, g, value=1.0 - self.beta2)
            denom = (v / bc2).sqrt_().add_(self.eps)
            p.addcdiv_(m, denom, value=-lrs[name] / bc1)


class TrainingDiverged(RuntimeError):
    """trainer.TrainingDiverged (trainer.py:172-173): the loss or a gradient
    of the step became non-finite."""

    def __init__(self, iteration: int, loss: float):
        super().__init__(f"training diverged at iteration {iteration}: loss {loss}")
        self.iteration, self.loss = iteration, loss


# --------------------------------------------------------------------------- sharding
def shard_views(batch: list, rank: int, world: int) -> list:
    """Round-robin assignment: batch position i goes to rank i mod world."""
    return [v for i, v in enumerate(batch) if i % world == rank]


class FlatGrads:
    """One contiguous float32 buffer: the six gradient tensors (pack_grads
    order of backward.py:322-329 per tensor) + sigma-signal sum + view count.
    A single all_reduce moves all of it."""

    def __init__(self, shapes: dict, n: int, device, dtype=torch.float32):
        self.names = list(PARAM_ORDER)
        sizes = [int(math.prod(shapes[k])) for k in self.names] + [n, n]
        self.buffer = torch.zeros(sum(sizes), dtype=dtype, device=device)
        self.views, off = {}, 0
        for k, sz in zip(self.names + ["sigma_signal", "sigma_views"], sizes):
            shape = shapes[k] if k in shapes else (n,)
            self.views[k] = self.buffer[off:off + sz].view(shape)
            off += sz

    def zero_(self):
        self.buffer.zero_()

    def grads(self) -> dict:
        return {k: self.views[k] for k in self.names}


class ViewShardedStep:
    """Training step over a batch of views, sharded across the ranks of
    ``group`` (world size 1 without torch.distributed).

    ``view_grad_fn(view, grads: dict, sigma_scratch) -> (loss, visible)``
    renders one view and ACCUMULATES its gradients into ``grads``; the default
    uses the sm_100a rasterizer and the device loss.  Tests substitute a CPU
    function to exercise the sharding / all-reduce / update logic under gloo.
    """

    def __init__(self, params: dict, config: StepConfig = StepConfig(), view_grad_fn: Callable = None,
                 group=None, buckets: int = 4):
        self.params = params
        self.config = config
        self.group = group
        self.distributed = dist.is_available() and dist.is_initialized()
        self.rank = dist.get_rank(group) if self.distributed else 0
        self.world = dist.get_world_size(group) if self.distributed else 1
        n = params["points"].shape[0]
        self.flat = FlatGrads({k: tuple(v.shape) for k, v in params.items()}, n, params["points"].device,
                              params["points"].dtype)
        if params["points"].device.type == "cuda":
            from .train_ops import FusedAdam
            self.adam = FusedAdam(params)      # one cs_adam_step launch for all six tensors
        else:
            self.adam = Adam(params)
        self.view_grad_fn = view_grad_fn
        self.iteration = 0
        # bucketed all-reduce: the rank's last view runs its
        # chain per convex range and each range's rows are all-reduced
        # (async) while the next range's chain runs; `buckets` ranges
        self.buckets = max(1, int(buckets))
        self._pending = []

    def lrs(self, iteration: int) -> dict:
        c = self.config
        return {"points": position_lr(iteration, c.lr_position_init, c.lr_position_final, c.total_iterations),
                "raw_delta": c.lr_delta, "raw_sigma": c.lr_sigma, "raw_opacity": c.lr_opacity, "sh": c.lr_sh,
                "raw_mask": c.lr_mask}

    def accumulate(self, batch: list) -> dict:
        """Local part: this rank's views, gradients summed into the flat buffer.
        A view function with ``handles_signal`` accumulates the per-view sigma
        signal itself (the CUDA path does it inside the backward's chain
        kernel); otherwise it is formed here from the gradient difference."""
        self.flat.zero_()
        grads = self.flat.grads()
        signal = {"sigma_signal": self.flat.views["sigma_signal"], "sigma_views": self.flat.views["sigma_views"]}
        own = getattr(self.view_grad_fn, "handles_signal", False)
        sigma_prev = None if own else torch.empty_like(grads["raw_sigma"])
        losses = []
        self._pending = []
        mine = shard_views(batch, self.rank, self.world)
        begin = getattr(self.view_grad_fn, "begin", None)
        if begin is not None:
            begin()
        bucketed = self.world > 1 and getattr(self.view_grad_fn, "supports_buckets", False)
        for vi, view in enumerate(mine):
            if own and bucketed and vi == len(mine) - 1:
                loss = self.view_grad_fn(view, grads, signal, ranges=self.bucket_ranges(),
                                         on_range=self._reduce_range)
            elif own:
                loss = self.view_grad_fn(view, grads, signal)
            else:
                sigma_prev.copy_(grads["raw_sigma"])
                loss, visible = self.view_grad_fn(view, grads)
                # trainer.py:192-193: per-view |d_raw_sigma| on the visible primitives
                vis = visible.to(self.flat.buffer.dtype)
                signal["sigma_signal"].add_((grads["raw_sigma"] - sigma_prev).abs_() * vis)
                signal["sigma_views"].add_(vis)
            losses.append(loss.detach().reshape(()))
        end = getattr(self.view_grad_fn, "end", None)
        if end is not None:
            end()
        losses = [x.to(self.flat.buffer.dtype) for x in losses]
        total = torch.stack(losses).sum() if losses else torch.zeros((), device=self.flat.buffer.device)
        return {"local_views": len(losses), "local_loss_sum": total}

    def bucket_ranges(self) -> list:
        n = self.flat.views["raw_delta"].shape[0]
        step = -(-n // self.buckets) if n else 1
        return [(i, min(i + step, n)) for i in range(0, n, step)]

    def _reduce_range(self, first: int, last: int):
        """All-reduce (async, SUM) of the rows [first, last) of every flat
        tensor: issued on NCCL's stream after the chain of that range, so it
        overlaps the chain of the next range."""
        for k in self.flat.views:
            self._pending.append(dist.all_reduce(self.flat.views[k][first:last], op=dist.ReduceOp.SUM,
                                                 group=self.group, async_op=True))

    def reduce(self, batch_size: int):
        """The collective: sum of everyone's gradients (the 1/B of the batch
        mean is applied inside the optimiser step) -- the bucketed
        all-reduces issued during the last view, or one all-reduce of the
        whole flat buffer."""
        if self.world <= 1:
            return
        if self._pending:
            for w in self._pending:
                w.wait()
            self._pending = []
        else:
            dist.all_reduce(self.flat.buffer, op=dist.ReduceOp.SUM, group=self.group)

    def step(self, batch: list) -> dict:
        self.iteration += 1
        info = self.accumulate(batch)
        check = getattr(self.view_grad_fn, "check_overflow", None)
        while check is not None and check(self.group if self.world > 1 else None):
            # a view of some rank overflowed its pair capacity: every rank redoes the step with more room
            for w in self._pending:
                w.wait()
            info = self.accumulate(batch)
        diverged = getattr(self.view_grad_fn, "diverged", None)
        if diverged is not None and diverged():   # trainer.py:172-173 (read with the overflow check)
            raise TrainingDiverged(self.iteration, float(info["local_loss_sum"]))
        self.reduce(len(batch))
        self.adam.step(self.params, self.flat.grads(), self.lrs(self.iteration), grad_scale=1.0 / len(batch))
        # densification signal since the last densify round (trainer.py:192-193)
        if not hasattr(self, "sigma_sum"):
            self.sigma_sum = torch.zeros_like(self.flat.views["sigma_signal"])
            self.sigma_views = torch.zeros_like(self.flat.views["sigma_views"])
        self.sigma_sum.add_(self.flat.views["sigma_signal"])
        self.sigma_views.add_(self.flat.views["sigma_views"])
        return info

    def densify(self, scene, density_config=None):
        """density.densify_and_prune on the device (trainer.py:195-203) with the
        accumulated signal sum / max(views, 1); identical on every rank (the
        signal was all-reduced).  Returns the new SceneTensors; ``params``, the
        Adam moments (remapped, optim.py:37-53), the flat buffers and the
        signal are rebuilt for it.  The caller re-creates its view function."""
        from .density import DensityConfig, densify_and_prune
        cfg = density_config or DensityConfig()
        signal = self.sigma_sum / torch.clamp(self.sigma_views, min=1.0)
        new, index_map, stats = densify_and_prune(scene, signal, cfg, self.iteration)
        self.params = {k: getattr(new, k) for k in PARAM_ORDER}
        self.adam.remap(index_map)
        n = new.n
        self.flat = FlatGrads({k: tuple(v.shape) for k, v in self.params.items()}, n, new.points.device,
                              new.points.dtype)
        self.sigma_sum = torch.zeros(n, dtype=self.flat.buffer.dtype, device=self.flat.buffer.device)
        self.sigma_views = torch.zeros_like(self.sigma_sum)
        self.last_densify = stats
        return new


def rasterizer_view_grad_fn(scene, mode, settings, config: StepConfig = StepConfig(), rasterizer=None,
                            lanes: int = 4):
    """Default per-view function on the GPU: sm_100a render, fused CUDA loss
    (cs_image_loss; adds the mask-loss gradient, trainer.py:176), backward
    through the C ABI accumulating into the flat buffers together with the
    view's sigma signal (cs_backward_signal).  Returns the view's loss as a
    device scalar.

    Views alternate between ``lanes`` CUDA streams, each with its own
    workspaces: the views of a step are independent until their gradients
    are summed (the backward's accumulation is by atomic reductions), so
    view v+1's forward overlaps view v's backward and the kernels' tails --
    every stage is latency-bound below full occupancy.  ViewShardedStep
    brackets a step's views with ``begin()`` / ``end()`` (fork from and join
    into the caller's stream).

    No host synchronisation per view: the forwards run with the cached pair
    capacity; each view's pair count and overflow flag are folded into a
    per-lane device maximum that ``check_overflow`` reads once per step -- if
    any view overflowed, the step is redone with a larger capacity."""
    from .rasterizer import Workspace, default_rasterizer
    from .train_ops import LossWorkspace, image_loss as cuda_image_loss

    r = rasterizer or default_rasterizer(scene.device)
    dev = scene.device
    n_lanes = max(1, int(os.environ.get("CS_VIEW_LANES", lanes)))   # (env: lane-count experiments)
    lane_state = [{"stream": torch.cuda.Stream(dev) if n_lanes > 1 else None, "ws": Workspace(dev),
                   "lw": LossWorkspace(),
                   # device maxima over the lane's views: (pairs, overflow, non-finite)
                   "max": torch.zeros(3, dtype=torch.int32, device=dev)} for _ in range(n_lanes)]
    state = {"cap": None, "bad": False, "next": 0, "forked": False}

    def begin():
        """Fork: every lane stream waits for the caller's stream (the zeroed
        flat buffer, the current parameters)."""
        state["next"] = 0
        if n_lanes > 1:
            ev = torch.cuda.current_stream(dev).record_event()
            for ln in lane_state:
                ln["stream"].wait_event(ev)
            state["forked"] = True

    def end():
        """Join: the caller's stream waits for every lane."""
        if n_lanes > 1 and state["forked"]:
            cur = torch.cuda.current_stream(dev)
            for ln in lane_state:
                cur.wait_stream(ln["stream"])
            state["forked"] = False

    def body(ln, view, grads, signal, ranges, on_range):
        cam, target = view
        ws, lw = ln["ws"], ln["lw"]
        if state["cap"] is None:      # first view ever: size the capacity with a checked forward
            fr = r.forward(scene, cam, mode, settings, workspace=ws, zero_accumulators=True)
            state["cap"] = fr.capacity
        else:   # the accumulator reset runs on a side stream under the forward
            fr = r.forward(scene, cam, mode, settings, workspace=ws, capacity=state["cap"], check=False,
                           zero_accumulators=True)
        torch.maximum(ln["max"][0:2], ws.counters()[1:3], out=ln["max"][0:2])   # (pairs, overflow)
        loss = cuda_image_loss(fr.image, target, scene.raw_mask, config.lambda_dssim, config.beta_mask,
                               d_raw_mask=grads["raw_mask"], workspace=lw)
        sig = (signal["sigma_signal"], signal["sigma_views"], fr.visible)
        if ranges is None:
            r.launch_backward(fr, loss["d_image"], grads, signal=sig)
        else:   # the chain per convex range, each range handed on as soon as it is final
            r.launch_backward(fr, loss["d_image"], grads, 0, 0)
            for first, last in ranges:
                r.launch_chain_range(fr, grads, first, last, signal=sig)
                on_range(first, last)
        # non-finite loss (trainer.py:172) or gradient row (the chain's C_NONFINITE flag)
        bad = (~torch.isfinite(loss["total"])).to(torch.int32).reshape(1)
        torch.maximum(ln["max"][2:3], torch.maximum(bad, ws.counters()[36:37]), out=ln["max"][2:3])
        return loss["total"]

    def fn(view, grads: dict, signal: dict, ranges=None, on_range=None):
        k = state["next"]
        state["next"] = k + 1
        ln = lane_state[k % n_lanes]
        if ln["stream"] is None or not state["forked"]:
            return body(ln, view, grads, signal, ranges, on_range)
        if ranges is not None:
            # the bucketed all-reduce reads rows the other lanes also add to:
            # this (last) view's lane first waits for them
            for other in lane_state:
                if other is not ln:
                    ln["stream"].wait_stream(other["stream"])
        with torch.cuda.stream(ln["stream"]):
            out = body(ln, view, grads, signal, ranges, on_range)
        out.record_stream(torch.cuda.current_stream(dev))
        return out

    def check_overflow(group=None) -> bool:
        """One host read per step: True (and a larger capacity) if any view
        overflowed its pair capacity since the last check -- on any rank of
        ``group`` (the maxima are all-reduced first), so that every rank
        redoes the step together."""
        mx = lane_state[0]["max"]
        for ln in lane_state[1:]:
            torch.maximum(mx, ln["max"], out=mx)
        if group is not None or (dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1):
            dist.all_reduce(mx, op=dist.ReduceOp.MAX, group=group)
        pairs, ovf, bad = (int(v) for v in mx.cpu())
        for ln in lane_state:
            ln["max"].zero_()
        state["bad"] = bool(bad) and not ovf
        if ovf:
            state["cap"] = int(pairs * 1.25) + 1024
            if state["cap"] >= (1 << 30):
                raise RuntimeError(f"{pairs} tile pairs exceed the supported 2^30")
            return True
        return False

    fn.handles_signal = True
    fn.supports_buckets = True
    fn.begin, fn.end = begin, end
    fn.check_overflow = check_overflow
    fn.diverged = lambda: state["bad"]
    return fn


def torch_view_grad_fn(scene, mode, settings, config: StepConfig = StepConfig(), rasterizer=None):
    """Per-view function with the loss formed by torch autograd of the
    losses.py expression (reference formulation; used by the tests)."""
    from .rasterizer import default_rasterizer

    r = rasterizer or default_rasterizer(scene.device)

    def fn(view, grads: dict):
        cam, target = view
        fr = r.forward(scene, cam, mode, settings)
        # the loss in float64, like the reference (float32 SSIM loses bits in
        # sxx = vxx - mu^2 on flat regions)
        img = fr.image.detach().double().requires_grad_(True)
        raw_mask = scene.raw_mask.detach().double().requires_grad_(True)
        loss = image_loss(img, target.double(), raw_mask, config.lambda_dssim, config.beta_mask)
        d_img, d_mask = torch.autograd.grad(loss["total"], (img, raw_mask))
        r.launch_backward(fr, d_img.float().contiguous(), grads)
        grads["raw_mask"].add_(d_mask.float())  # trainer.py:176 (straight-through mask-loss term)
        return loss["total"].detach().float(), fr.visible
    return fn


__all__ = ["StepConfig", "TrainingDiverged", "image_loss", "ssim", "gaussian_window", "Adam", "position_lr", "shard_views",
           "FlatGrads", "ViewShardedStep", "rasterizer_view_grad_fn", "torch_view_grad_fn"]
