"""Host side of the sm_100a rasterizer: workspace management, the autograd
Function and the reference-compatible entry points.

Layering (north_star): Python API with the reference names
(rasterize.render / render_reference / prepare_view / bin_tiles,
backward.backward) -> torch.autograd.Function -> ctypes ->
libconvexsplat_sm100.so (extern "C", include/convexsplat_b200.h) -> kernels.
There is no CPU path: every call goes through the CUDA library and raises if
it is unavailable.
"""
from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field
from typing import Optional

import numpy as np
import torch

from . import _lib
from .model import (EXACT_SETTINGS, SH_COEFFS, Camera, GradientBuffer, RenderOutput,
                    RenderSettings, ScalingMode)
from .scene_tensors import SceneTensors, as_scene_tensors

_COUNTERS = 40
STAT_NAMES = ("fwd_evals", "fwd_line_evals", "fwd_blends", "bwd_evals", "bwd_line_evals", "fwd_warp_evals",
              "bwd_warp_evals", "bwd_blends")


def _device(device=None) -> torch.device:
    if not torch.cuda.is_available():
        raise _lib.CsError("the convex-splatting renderer needs a CUDA device (no CPU fallback)")
    if device is None:
        return torch.device("cuda", torch.cuda.current_device())
    device = torch.device(device)
    if device.type != "cuda":
        raise _lib.CsError(f"the renderer runs on CUDA devices only, got {device}")
    return torch.device("cuda", device.index if device.index is not None else torch.cuda.current_device())


def camera_struct(cam: Camera) -> _lib.CsCamera:
    c = _lib.CsCamera()
    c.fx, c.fy, c.cx, c.cy = float(cam.fx), float(cam.fy), float(cam.cx), float(cam.cy)
    c.R[:] = [float(v) for v in np.asarray(cam.R, dtype=np.float64).reshape(9)]
    c.t[:] = [float(v) for v in np.asarray(cam.t, dtype=np.float64).reshape(3)]
    c.z_near = float(cam.z_near)
    c.width, c.height = int(cam.width), int(cam.height)
    c.ortho = int(bool(cam.ortho))
    return c


def settings_struct(settings: RenderSettings, mode: ScalingMode, background) -> _lib.CsSettings:
    s = _lib.CsSettings()
    s.cutoff = float(settings.contribution_cutoff)
    s.floor = float(settings.transmittance_floor)
    s.background[:] = [float(v) for v in np.asarray(background, dtype=np.float64).reshape(3)]
    s.tile = int(settings.tile_size)
    s.sh_degree = int(settings.sh_degree)
    s.scaling_mode = ScalingMode.of(mode).code
    return s


def params_struct(st: SceneTensors) -> _lib.CsParams:
    for name in ("points", "raw_delta", "raw_sigma", "raw_opacity", "raw_mask", "sh"):
        t = getattr(st, name)
        if t.dtype != torch.float32 or not t.is_contiguous() or t.device.type != "cuda":
            raise ValueError(f"{name} must be a contiguous float32 CUDA tensor")
    p = _lib.CsParams()
    p.n, p.k = st.n, st.k
    p.points, p.raw_delta, p.raw_sigma = st.points.data_ptr(), st.raw_delta.data_ptr(), st.raw_sigma.data_ptr()
    p.raw_opacity, p.raw_mask, p.sh = st.raw_opacity.data_ptr(), st.raw_mask.data_ptr(), st.sh.data_ptr()
    return p


class Workspace:
    """Caller-owned device workspace of one frame (the C ABI never allocates)."""

    def __init__(self, device=None):
        self.device = _device(device)
        self.buffer: Optional[torch.Tensor] = None
        self.layout: Optional[_lib.CsLayout] = None
        self.capacity = 0

    def plan(self, cam_c, set_c, n: int, k: int, capacity: int) -> _lib.CsLayout:
        L = _lib.CsLayout()
        _lib.check(_lib.load().cs_workspace_layout(ctypes.byref(cam_c), ctypes.byref(set_c), n, k, capacity,
                                                   ctypes.byref(L)), "cs_workspace_layout")
        return L

    def ensure(self, cam_c, set_c, n: int, k: int, capacity: int) -> _lib.CsLayout:
        L = self.plan(cam_c, set_c, n, k, capacity)
        if self.buffer is None or self.buffer.numel() < L.total_bytes:
            self.buffer = torch.empty(int(L.total_bytes * 1.05) + 256, dtype=torch.uint8, device=self.device)
        self.layout, self.capacity = L, capacity
        return L

    @property
    def ptr(self) -> int:
        return self.buffer.data_ptr()

    @property
    def nbytes(self) -> int:
        return self.buffer.numel()

    def region(self, name: str, dtype: torch.dtype, count: int) -> torch.Tensor:
        off = getattr(self.layout, name)
        nbytes = count * torch.empty((), dtype=dtype).element_size()
        return self.buffer[off:off + nbytes].view(dtype)

    def counters(self) -> torch.Tensor:
        return self.region("counters", torch.int32, _COUNTERS)


@dataclass
class Frame:
    """Result of one forward render (device tensors) + what the backward needs."""

    image: torch.Tensor
    final_T: torch.Tensor
    count: torch.Tensor
    weight_sum: torch.Tensor
    depth: torch.Tensor
    visible: torch.Tensor
    workspace: Workspace
    scene: SceneTensors
    cam_c: _lib.CsCamera
    set_c: _lib.CsSettings
    params_c: _lib.CsParams
    capacity: int
    n_visible: int = -1
    n_pairs: int = -1
    extras: dict = field(default_factory=dict)


class Rasterizer:
    """Stateless apart from a pair-capacity hint; each forward gets its own
    workspace unless one is passed (the benchmark reuses one)."""

    def __init__(self, device=None, growth: float = 1.25):
        self.device = _device(device)
        self.growth = growth
        self._cap_hint = {}
        self._side_streams = {}
        _lib.load()

    def _initial_capacity(self, st: SceneTensors, cam: Camera) -> int:
        key = (st.n, cam.width, cam.height)
        if key in self._cap_hint:
            return self._cap_hint[key]
        tiles = math.ceil(cam.width / 16) * math.ceil(cam.height / 16)
        return int(min(max(8 * st.n, 4096), max(st.n * tiles, 4096), (1 << 30) - 1))

    def forward(self, scene, cam: Camera, mode=ScalingMode.DEPTH, settings: RenderSettings = RenderSettings(),
                workspace: Optional[Workspace] = None, capacity: Optional[int] = None, check: bool = True,
                outputs: Optional[dict] = None, zero_accumulators: bool = False) -> Frame:
        """Render (cs_forward).  ``check``: read the pair count back and
        re-render with a larger capacity on overflow (one host sync).
        ``zero_accumulators``: also reset the backward accumulators on a side
        stream (``zero_accumulators_async``; overlapping the forward when
        ``check`` is off)."""
        st = as_scene_tensors(scene, self.device)
        cam_c = camera_struct(cam)
        set_c = settings_struct(settings, mode, st.background)
        params_c = params_struct(st)
        ws = workspace if workspace is not None else Workspace(self.device)
        cap = capacity if capacity is not None else max(ws.capacity, self._initial_capacity(st, cam))
        H, W, n = cam.height, cam.width, st.n
        if outputs is None:
            dev = self.device
            outputs = dict(image=torch.empty((H, W, 3), device=dev), final_T=torch.empty((H, W), device=dev),
                           count=torch.empty((H, W), dtype=torch.int32, device=dev),
                           weight_sum=torch.empty((H, W), device=dev), depth=torch.empty((H, W), device=dev),
                           visible=torch.empty((max(n, 1),), dtype=torch.uint8, device=dev))
        frame_c = _lib.CsFrame(outputs["image"].data_ptr(), outputs["final_T"].data_ptr(),
                               outputs["count"].data_ptr(), outputs["weight_sum"].data_ptr(),
                               outputs["depth"].data_ptr(), outputs["visible"].data_ptr())
        stream = torch.cuda.current_stream(self.device).cuda_stream
        while True:
            ws.ensure(cam_c, set_c, n, st.k, cap)
            zeroed = self._fork_zero(cam_c, set_c, params_c, ws, cap) if zero_accumulators and not check else None
            _lib.check(_lib.load().cs_forward(ctypes.byref(cam_c), ctypes.byref(set_c), ctypes.byref(params_c),
                                              ws.ptr, ws.nbytes, cap, ctypes.byref(frame_c), stream), "cs_forward")
            fr = Frame(outputs["image"], outputs["final_T"], outputs["count"], outputs["weight_sum"],
                       outputs["depth"], outputs["visible"][:n], ws, st, cam_c, set_c, params_c, cap)
            fr.extras["frame_c"] = frame_c
            if not check:
                if zeroed is not None:
                    fr.extras["accum_zeroed"] = zeroed
                return fr
            counts = (ctypes.c_uint32 * 4)()
            _lib.check(_lib.load().cs_read_counters(ctypes.c_void_p(ws.ptr), counts, stream), "cs_read_counters")
            fr.n_visible, fr.n_pairs = int(counts[0]), int(counts[1])
            if counts[2] == 0:
                self._cap_hint[(n, W, H)] = max(cap, int(fr.n_pairs * self.growth) + 1024)
                if zero_accumulators:
                    self.zero_accumulators_async(fr)
                return fr
            cap = int(fr.n_pairs * self.growth) + 1024   # overflow: grow and re-render
            if cap >= (1 << 30):
                raise _lib.CsError(f"{fr.n_pairs} tile pairs exceed the supported 2^30")

    def _fork_zero(self, cam_c, set_c, params_c, ws, cap) -> torch.cuda.Event:
        cur = torch.cuda.current_stream(self.device)
        side = self._side_streams.get(cur.cuda_stream)
        if side is None:   # one side stream per issuing stream (view lanes run concurrently)
            side = self._side_streams[cur.cuda_stream] = torch.cuda.Stream(self.device)
        fork = torch.cuda.Event()
        fork.record(cur)
        side.wait_event(fork)
        _lib.check(_lib.load().cs_zero_accumulators(ctypes.byref(cam_c), ctypes.byref(set_c), ctypes.byref(params_c),
                                                    ws.ptr, ws.nbytes, cap, side.cuda_stream), "cs_zero_accumulators")
        done = torch.cuda.Event()
        done.record(side)
        return done

    def zero_accumulators_async(self, fr: Frame):
        """Reset ``fr``'s backward accumulators on a side stream, forked from
        the current stream now (after everything already queued on it, e.g.
        the previous chain that read them); the next ``launch_backward`` of
        the frame joins it and skips its own reset (CS_ACCUM_ZEROED).  Issued
        before the forward's launches, the 256 MB reset (1M convexes) runs
        under the latency-bound forward kernels instead of after them."""
        fr.extras["accum_zeroed"] = self._fork_zero(fr.cam_c, fr.set_c, fr.params_c, fr.workspace, fr.capacity)

    def launch_forward(self, fr: Frame, first_stage: int = 0, last_stage: int = 2, work_counters: bool = False,
                       zero_accumulators: bool = False):
        """Re-run forward stages of an existing frame (same scene tensors,
        camera, workspace and outputs) without any host synchronisation;
        stages: 0 preprocess, 1 depth order + binning, 2 blend.
        ``work_counters``: the blend also counts its work (``read_stats``).
        ``zero_accumulators``: reset the backward accumulators alongside
        (``zero_accumulators_async``)."""
        if zero_accumulators:
            self.zero_accumulators_async(fr)
        ws = fr.workspace
        stream = torch.cuda.current_stream(self.device).cuda_stream
        _lib.check(_lib.load().cs_forward_ex(ctypes.byref(fr.cam_c), ctypes.byref(fr.set_c),
                                             ctypes.byref(fr.params_c), ws.ptr, ws.nbytes, fr.capacity,
                                             ctypes.byref(fr.extras["frame_c"]),
                                             _lib.WORK_COUNTERS if work_counters else 0, first_stage, last_stage,
                                             stream), "cs_forward_ex")

    def launch_backward(self, fr: Frame, d_image: torch.Tensor, grads: dict, first_stage: int = 0,
                        last_stage: int = 1, signal=None, overwrite: bool = False, work_counters: bool = False):
        """Backward stages (0 blend, 1 chain) into ``grads`` (+=, or written
        when ``overwrite``: every row, zeros for convexes the view did not
        prepare), no sync.  ``signal`` = (sigma_signal, sigma_views, visible)
        tensors: also accumulate the view's densification signal
        (trainer.py:192-193)."""
        g = _lib.CsGrads(grads["points"].data_ptr(), grads["raw_delta"].data_ptr(), grads["raw_sigma"].data_ptr(),
                         grads["raw_opacity"].data_ptr(), grads["raw_mask"].data_ptr(), grads["sh"].data_ptr())
        ws = fr.workspace
        cur = torch.cuda.current_stream(self.device)
        stream = cur.cuda_stream
        zeroed = 0
        if first_stage == 0:
            ev = fr.extras.pop("accum_zeroed", None)
            if ev is not None:      # the reset forked by zero_accumulators_async
                cur.wait_event(ev)
                zeroed = _lib.ACCUM_ZEROED
        sig = None
        if signal is not None:
            if (first_stage, last_stage) != (0, 1):
                raise ValueError("the sigma signal needs the full backward")
            sig = _lib.CsViewSignal(signal[0].data_ptr(), signal[1].data_ptr(), signal[2].data_ptr())
        _lib.check(_lib.load().cs_backward_ex(ctypes.byref(fr.cam_c), ctypes.byref(fr.set_c),
                                              ctypes.byref(fr.params_c), ws.ptr, ws.nbytes, fr.capacity,
                                              d_image.data_ptr(), ctypes.byref(g),
                                              ctypes.byref(sig) if sig is not None else None,
                                              (_lib.GRADS_OVERWRITE if overwrite else 0) |
                                              (_lib.WORK_COUNTERS if work_counters else 0) | zeroed, first_stage,
                                              last_stage, stream), "cs_backward_ex")

    def launch_chain_range(self, fr: Frame, grads: dict, first: int, last: int, signal=None):
        """Stage 1 (the per-convex chain) of a backward whose stage 0 ran,
        over convexes [first, last) only, accumulating (+=) into ``grads``
        (cs_backward_chain_range): the bucketed all-reduce of the
        view-sharded step starts on a range as soon as its chain is done."""
        g = _lib.CsGrads(grads["points"].data_ptr(), grads["raw_delta"].data_ptr(), grads["raw_sigma"].data_ptr(),
                         grads["raw_opacity"].data_ptr(), grads["raw_mask"].data_ptr(), grads["sh"].data_ptr())
        ws = fr.workspace
        sig = None
        if signal is not None:
            sig = _lib.CsViewSignal(signal[0].data_ptr(), signal[1].data_ptr(), signal[2].data_ptr())
        stream = torch.cuda.current_stream(self.device).cuda_stream
        _lib.check(_lib.load().cs_backward_chain_range(ctypes.byref(fr.cam_c), ctypes.byref(fr.set_c),
                                                       ctypes.byref(fr.params_c), ws.ptr, ws.nbytes, fr.capacity,
                                                       ctypes.byref(g), ctypes.byref(sig) if sig is not None else None,
                                                       0, int(first), int(last), stream), "cs_backward_chain_range")

    @staticmethod
    def read_stats(fr: Frame) -> dict:
        """Work counters of the last forward/backward on this workspace (syncs);
        the blend counts are filled only by calls with ``work_counters``."""
        c = fr.workspace.counters().cpu()
        stats = c[16:32].view(torch.int64).numpy()
        out = {name: int(stats[i]) for i, name in enumerate(STAT_NAMES)}
        out.update(n_visible=int(c[0]), n_pairs=int(c[1]), overflow=int(c[2]), nonfinite=int(c[36]))
        return out

    def status(self, fr: Frame) -> int:
        """cs_read_status of the frame's workspace (syncs): 0 ok,
        _lib.ERR_NONFINITE when the last backward produced an inf/NaN
        gradient row, _lib.ERR_WORKSPACE when the pairs overflowed."""
        stream = torch.cuda.current_stream(self.device).cuda_stream
        return int(_lib.load().cs_read_status(fr.workspace.ptr, stream))

    def backward(self, frame: Frame, d_image: torch.Tensor, grads: dict, overwrite: bool = False) -> dict:
        """Accumulate (+=) gradients of sum(d_image * image) into ``grads``,
        or write them (``overwrite``: ``grads`` may be uninitialised)."""
        d_image = d_image.to(device=self.device, dtype=torch.float32).contiguous()
        H, W = frame.cam_c.height, frame.cam_c.width
        if tuple(d_image.shape) != (H, W, 3):
            raise ValueError(f"d_image must be ({H}, {W}, 3), got {tuple(d_image.shape)}")
        self.launch_backward(frame, d_image, grads, overwrite=overwrite)
        return grads


def zero_grads(st: SceneTensors) -> dict:
    return {name: torch.zeros_like(getattr(st, name)) for name in
            ("points", "raw_delta", "raw_sigma", "raw_opacity", "raw_mask", "sh")}


def empty_grads(st: SceneTensors) -> dict:
    """Uninitialised gradient buffers for an overwriting backward."""
    return {name: torch.empty_like(getattr(st, name)) for name in
            ("points", "raw_delta", "raw_sigma", "raw_opacity", "raw_mask", "sh")}


_default: dict = {}


def default_rasterizer(device=None) -> Rasterizer:
    dev = _device(device)
    if dev not in _default:
        _default[dev] = Rasterizer(dev)
    return _default[dev]


# ---------------------------------------------------------------------------
# autograd


class _RasterizeFunction(torch.autograd.Function):
    @staticmethod
    def forward(ctx, rasterizer, cam, mode, settings, background, points, raw_delta, raw_sigma, raw_opacity,
                raw_mask, sh):
        st = SceneTensors(points.detach().contiguous(), raw_delta.detach().contiguous(),
                          raw_sigma.detach().contiguous(), raw_opacity.detach().contiguous(),
                          raw_mask.detach().contiguous(), sh.detach().contiguous(), background)
        # a backward will follow: its accumulator reset runs on a side stream now
        fr = rasterizer.forward(st, cam, mode, settings, zero_accumulators=any(ctx.needs_input_grad[5:]))
        ctx.frame, ctx.rasterizer = fr, rasterizer
        ctx.mark_non_differentiable(fr.final_T, fr.count, fr.weight_sum, fr.depth, fr.visible)
        return fr.image, fr.final_T, fr.count, fr.weight_sum, fr.depth, fr.visible

    @staticmethod
    def backward(ctx, d_image, *_unused):
        fr = ctx.frame
        if d_image is not None:
            grads = ctx.rasterizer.backward(fr, d_image, empty_grads(fr.scene), overwrite=True)
        else:
            grads = zero_grads(fr.scene)
        ctx.frame = None
        return (None, None, None, None, None, grads["points"], grads["raw_delta"], grads["raw_sigma"],
                grads["raw_opacity"], grads["raw_mask"], grads["sh"])


def rasterize(scene: SceneTensors, cam: Camera, mode=ScalingMode.DEPTH, settings: RenderSettings = RenderSettings(),
              rasterizer: Optional[Rasterizer] = None):
    """Differentiable render of SoA tensors.  Returns (image, final_T, count,
    weight_sum, depth, visible); gradients flow from ``image`` to the six
    parameter tensors (backward.py:76-282 semantics)."""
    r = rasterizer or default_rasterizer(scene.device)
    return _RasterizeFunction.apply(r, cam, mode, settings, scene.background, scene.points, scene.raw_delta,
                                    scene.raw_sigma, scene.raw_opacity, scene.raw_mask, scene.sh)


# ---------------------------------------------------------------------------
# reference-compatible entry points (numpy in/out, float64 like the reference)


def _np(t: torch.Tensor) -> np.ndarray:
    return t.detach().cpu().numpy()


def render(scene, cam: Camera, mode: ScalingMode = ScalingMode.DEPTH,
           settings: RenderSettings = RenderSettings()) -> RenderOutput:
    """rasterize.render (rasterize.py:156-209) on the GPU."""
    fr = default_rasterizer().forward(scene, cam, mode, settings)
    return RenderOutput(image=_np(fr.image).astype(np.float64),
                        final_transmittance=_np(fr.final_T).astype(np.float64),
                        per_pixel_count=_np(fr.count), blend_weight_sum=_np(fr.weight_sum).astype(np.float64),
                        visible=_np(fr.visible).astype(bool), depth=_np(fr.depth).astype(np.float64))


def render_reference(scene, cam: Camera, mode: ScalingMode = ScalingMode.DEPTH) -> RenderOutput:
    """rasterize.render_reference (rasterize.py:212-245): every primitive at
    every pixel with no bbox, cutoff or termination -- identical semantics to
    render(EXACT_SETTINGS) (test_rasterize.py:118-128), so it runs the same
    kernels with full-frame bboxes."""
    return render(scene, cam, mode, EXACT_SETTINGS)


def backward(scene, cam: Camera, d_image, mode: ScalingMode = ScalingMode.DEPTH,
             settings: RenderSettings = RenderSettings()) -> GradientBuffer:
    """backward.backward (backward.py:76-212): gradient of sum(d_image*image)."""
    r = default_rasterizer()
    st = as_scene_tensors(scene, r.device)
    fr = r.forward(st, cam, mode, settings)
    grads = r.backward(fr, torch.as_tensor(np.asarray(d_image), dtype=torch.float32), empty_grads(st), overwrite=True)
    f64 = {k: _np(v).astype(np.float64) for k, v in grads.items()}
    return GradientBuffer(d_points=f64["points"], d_raw_delta=f64["raw_delta"], d_raw_sigma=f64["raw_sigma"],
                          d_raw_opacity=f64["raw_opacity"], d_sh=f64["sh"], d_raw_mask=f64["raw_mask"],
                          visible=_np(fr.visible).astype(bool))


# ---------------------------------------------------------------------------
# discrete state of a frame (prepare_view / bin_tiles equivalents)


def _decode_depth(keys: np.ndarray) -> np.ndarray:
    """Inverse of the order-preserving f64 -> u64 map of csrc/common.cuh."""
    keys = keys.astype(np.uint64)
    sign = (keys & np.uint64(1 << 63)) != 0
    bits = np.where(sign, keys & ~np.uint64(1 << 63), ~keys)
    return bits.view(np.float64)


def inspect_frame(fr: Frame) -> dict:
    """Copy the frame's discrete state to host: depth order, hull cycles,
    bboxes and the per-tile candidate lists (CSR over row-major tiles)."""
    ws, L = fr.workspace, fr.workspace.layout
    n, V, P = fr.scene.n, fr.n_visible, fr.n_pairs
    tiles = L.tiles_x * L.tiles_y
    order = _np(ws.region("order", torch.int32, n))[:V].astype(np.int64)
    hull = _np(ws.region("hull", torch.uint8, n * L.max_k)).reshape(n, L.max_k).astype(np.int64)
    hull[hull == 255] = -1
    bbox = _np(ws.region("bbox", torch.int32, 4 * n)).reshape(n, 4).astype(np.int64)
    keys = _np(ws.region("depth_keys", torch.int64, n)).view(np.uint64)[order]
    ranges = _np(ws.region("tile_ranges", torch.int32, 2 * tiles)).reshape(tiles, 2).astype(np.int64)
    pair_ids = _np(ws.region("pair_ids", torch.int32, P)).astype(np.int64)
    recs = _np(ws.region("records", torch.float32, n * L.rec_floats)).reshape(n, L.rec_floats)
    off = np.zeros(tiles + 1, np.int64)
    counts = np.zeros(tiles, np.int64)
    nz = ranges[:, 1] > ranges[:, 0]
    counts[nz] = ranges[nz, 1] - ranges[nz, 0]
    off[1:] = np.cumsum(counts)
    # tile of every list entry (CSR order)
    pair_tiles = np.repeat(np.arange(tiles, dtype=np.int64), counts)
    return dict(order=order, hull=hull, bbox=bbox, depth=_decode_depth(keys), tile_ranges=ranges,
                pair_ids=pair_ids, pair_tiles=pair_tiles, tile_offsets=off, records=recs,
                tiles_x=L.tiles_x, tiles_y=L.tiles_y, n_visible=V, n_pairs=P)


def record_blends(fr: Frame):
    """The frame's blend decisions (diagnostics for the decision-forced
    parity check, cs_forward_record): (offsets [H*W+1] int64, positions
    int32 -- pixel p blended the pair indices positions[offsets[p]:
    offsets[p+1]] in blend order --, clamp [H*W] uint8 -- bit c set iff
    channel c of C + T*bg lay in [0, 1], the clip test of
    backward.py:154-158).  Re-runs the frame's blend stage with the same
    kernel (it is deterministic) while recording."""
    ws, L = fr.workspace, fr.workspace.layout
    H, W = fr.cam_c.height, fr.cam_c.width
    counts = fr.count.reshape(-1).to(torch.int64)
    offsets = torch.zeros(H * W + 1, dtype=torch.int64, device=counts.device)
    torch.cumsum(counts, 0, out=offsets[1:])
    total = int(offsets[-1])
    pos = torch.full((max(total, 1),), -1, dtype=torch.int32, device=counts.device)
    starts = offsets[:-1].contiguous()
    count0 = fr.count.clone()
    stream = torch.cuda.current_stream(counts.device).cuda_stream
    _lib.check(_lib.load().cs_forward_record(ctypes.byref(fr.cam_c), ctypes.byref(fr.set_c),
                                             ctypes.byref(fr.params_c), ws.ptr, ws.nbytes, fr.capacity,
                                             ctypes.byref(fr.extras["frame_c"]), starts.data_ptr(),
                                             pos.data_ptr(), stream), "cs_forward_record")
    if not torch.equal(fr.count, count0):
        raise _lib.CsError("cs_forward_record: the re-run blend decided differently")
    clamp = ws.region("pixel_clamp", torch.uint8, H * W)
    return _np(offsets), _np(pos)[:total], _np(clamp)


@dataclass
class ProjectedConvex:
    """projection.ProjectedConvex (projection.py:180-203): per-view
    screen-space state of one primitive, float64 (cs_prepare_view_export)."""

    index: int
    pixels: np.ndarray        # (K, 2)
    point_depths: np.ndarray  # (K,)
    depth: float
    hull_indices: np.ndarray  # (H,)
    normals: np.ndarray       # (H, 2)
    offsets: np.ndarray       # (H,)
    delta_s: float
    sigma_s: float
    bbox: tuple               # (x0, x1, y0, y1) half-open pixel rect

    @property
    def hull_pixels(self) -> np.ndarray:
        return self.pixels[self.hull_indices]


@dataclass
class ViewPrimitive:
    """rasterize.ViewPrimitive (rasterize.py:56-65)."""

    pc: ProjectedConvex
    opacity: float
    color: np.ndarray
    scale: float           # depth scale applied to delta and sigma
    view_dir: np.ndarray   # unit vector camera center -> primitive center
    view_dist: float


class PreparedView(list):
    """prepare_view() result: ViewPrimitives in blend order + the GPU tile lists."""

    bins: list = None
    tiles_x: int = 0
    tiles_y: int = 0


def prepare_view(scene, cam: Camera, mode: ScalingMode = ScalingMode.DEPTH,
                 settings: RenderSettings = RenderSettings()) -> PreparedView:
    """rasterize.prepare_view (rasterize.py:77-122) from the GPU preprocess:
    the visible primitives in blending order (depth, index) with the float64
    per-view state of cs_prepare_view_export; ``bins`` holds the GPU tile
    lists (bin_tiles)."""
    r = default_rasterizer()
    fr = r.forward(scene, cam, mode, settings)
    info = inspect_frame(fr)
    st, dev = fr.scene, fr.image.device
    n, k = st.n, st.k
    f64 = dict(dtype=torch.float64, device=dev)
    ex = {"pixels": torch.zeros((n, k, 2), **f64), "point_depths": torch.zeros((n, k), **f64),
          "normals": torch.zeros((n, k, 2), **f64), "offsets": torch.zeros((n, k), **f64),
          "delta_s": torch.zeros(n, **f64), "sigma_s": torch.zeros(n, **f64), "opacity": torch.zeros(n, **f64),
          "scale": torch.zeros(n, **f64), "view_dir": torch.zeros((n, 3), **f64), "view_dist": torch.zeros(n, **f64),
          "color": torch.zeros((n, 3), **f64)}
    out_c = _lib.CsViewExport(*(ex[f].data_ptr() for f, _ in _lib.CsViewExport._fields_))
    ws = fr.workspace
    _lib.check(_lib.load().cs_prepare_view_export(ctypes.byref(fr.cam_c), ctypes.byref(fr.set_c),
                                                  ctypes.byref(fr.params_c), ws.ptr, ws.nbytes, fr.capacity,
                                                  ctypes.byref(out_c), torch.cuda.current_stream(dev).cuda_stream),
               "cs_prepare_view_export")
    ex = {f: _np(v) for f, v in ex.items()}
    out = PreparedView()
    for rank, i in enumerate(info["order"]):
        h = info["hull"][i]
        h = h[h >= 0].copy()
        nh = h.size
        pc = ProjectedConvex(int(i), ex["pixels"][i].copy(), ex["point_depths"][i].copy(), float(info["depth"][rank]),
                             h, ex["normals"][i, :nh].copy(), ex["offsets"][i, :nh].copy(), float(ex["delta_s"][i]),
                             float(ex["sigma_s"][i]), tuple(int(v) for v in info["bbox"][i]))
        out.append(ViewPrimitive(pc, float(ex["opacity"][i]), ex["color"][i].copy(), float(ex["scale"][i]),
                                 ex["view_dir"][i].copy(), float(ex["view_dist"][i])))
    rank_of = np.full(n, -1, np.int64)
    rank_of[info["order"]] = np.arange(len(info["order"]))
    bins = []
    for t in range(info["tiles_x"] * info["tiles_y"]):
        s0, e = info["tile_ranges"][t]
        bins.append(rank_of[info["pair_ids"][s0:e]].tolist() if e > s0 else [])
    out.bins, out.tiles_x, out.tiles_y = bins, info["tiles_x"], info["tiles_y"]
    return out


def bin_tiles(prepared, width: int, height: int, tile_size: int = 16):
    """rasterize.bin_tiles (rasterize.py:134-144): per-tile candidate lists of
    positions in the prepared order, row-major tiles; returns (bins,
    tiles_x, tiles_y).  For this package's prepare_view() result these are
    the GPU binning's lists; for any other prepared list (e.g. the
    reference's own ViewPrimitives) the (tile, position) pairs of the
    ``pc.bbox`` rectangles are expanded and stably sorted by tile on the
    GPU."""
    tiles_x = (width + tile_size - 1) // tile_size
    tiles_y = (height + tile_size - 1) // tile_size
    if isinstance(prepared, PreparedView) and prepared.bins is not None and tile_size == 16 \
            and (tiles_x, tiles_y) == (prepared.tiles_x, prepared.tiles_y):
        return [list(b) for b in prepared.bins], tiles_x, tiles_y
    bins = [[] for _ in range(tiles_x * tiles_y)]
    if len(prepared) == 0:
        return bins, tiles_x, tiles_y
    dev = _device()
    bb = torch.tensor([tuple(vp.pc.bbox) for vp in prepared], dtype=torch.int64, device=dev)
    tx0, tx1 = bb[:, 0] // tile_size, (bb[:, 1] - 1) // tile_size
    ty0, ty1 = bb[:, 2] // tile_size, (bb[:, 3] - 1) // tile_size
    nx, ny = tx1 - tx0 + 1, ty1 - ty0 + 1
    cnt = nx * ny
    pos = torch.repeat_interleave(torch.arange(len(prepared), device=dev), cnt)
    start = torch.cumsum(cnt, 0) - cnt
    j = torch.arange(int(cnt.sum()), device=dev) - torch.repeat_interleave(start, cnt)
    tile = (ty0[pos] + j // nx[pos]) * tiles_x + tx0[pos] + j % nx[pos]
    tile_sorted, perm = torch.sort(tile, stable=True)       # position order kept within a tile
    counts = torch.bincount(tile_sorted, minlength=tiles_x * tiles_y).cpu().tolist()
    flat = pos[perm].cpu().tolist()
    o = 0
    for t, c in enumerate(counts):
        bins[t] = flat[o:o + c]
        o += c
    return bins, tiles_x, tiles_y


__all__ = ["Rasterizer", "Workspace", "Frame", "rasterize", "render", "render_reference", "backward",
           "prepare_view", "bin_tiles", "inspect_frame", "zero_grads", "empty_grads", "default_rasterizer",
           "camera_struct", "settings_struct", "params_struct", "SH_COEFFS"]
