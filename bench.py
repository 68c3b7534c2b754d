#!/usr/bin/env python
"""Benchmark of the sm_100a convex-splatting hot path (BASELINE.json metric).

Headline workload (BASELINE.json configs[3]): G(1M, seed 0)
six-point convexes, camera C(1920, 1080), DEPTH scaling, RenderSettings()
defaults, synthetic float32 scene (no dataset), d_image ~ N(0, 1e-3) for the
backward.

* ``value``: forward frames/s over all ranks (each rank renders a replica of
  the single view: one view is not partitioned), scene resident
  in HBM, L2 flushed before every timed frame (a 512 MB write, untimed).
* ``fwd_bwd_iters_per_s``: forward + backward (fresh gradients).
* ``e2e``: same metric through the C-ABI call with HOST buffers: pinned
  host->device copy of the six parameter arrays, cs_forward, device->host
  copy of the image, all inside the timed region.
* ``roofline``: the dominant kernel of the fwd+bwd frame, with SURVEY 8(d)'s
  algorithmic work per stage (``roofline.stages``) and the frame composites
  sum(t_ideal) / t_frame.
* ``configs``: BASELINE.json configs 1-3 (1k @256^2 fwd+bwd on the
  reference's own config-1 scene; the toy-chair fit, 128 views @512^2 per
  training step; 100k @1297x840 forward), each with the CPU reference path
  timed beside it (N = 1 only).
* ``train_step``: config 5, the view-sharded training step (64 views
  1297x840, NCCL all_reduce of the gradients) on all ranks.
* ``cpu_baseline``: the float64 C oracle (port of the reference, oracle/)
  on this box's host cores over a bounded sample of tiles.

``--gpus N`` without a torchrun environment re-launches itself under
``torch.distributed.run`` with N ranks (127.0.0.1 rendezvous).
``--impl reference`` times only the CPU reference path (the oracle port) on
the host cores and prints the same JSON line with ``"impl": "reference"``.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "fwd FPS & fwd+bwd iters/s, 1M 6-pt convexes @1080p; % of roofline"
UNIT = "frames/s"
MUFU_PER_CLK_PER_SM = 16     # CUDA arithmetic-throughput table, sm_100
N_SMS = 148


def parse_args():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", choices=("ours", "reference"), default="ours")
    p.add_argument("--n", type=int, default=1_000_000)
    p.add_argument("--width", type=int, default=1920)
    p.add_argument("--height", type=int, default=1080)
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--cpu-budget-s", type=float, default=15.0, help="CPU-baseline sample budget")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-train", action="store_true", help="skip the config-5 view-sharded training step")
    p.add_argument("--no-configs", action="store_true", help="skip the config 1-3 blocks")
    p.add_argument("--cpu-check", action="store_true",
                   help="launcher / collective check without a GPU: the config-5 step logic on CPU over gloo")
    p.add_argument("--chair-views", type=int, default=128)
    p.add_argument("--chair-size", type=int, default=512)
    p.add_argument("--chair-steps", type=int, default=3)
    p.add_argument("--train-views", type=int, default=64)
    p.add_argument("--train-width", type=int, default=1297)
    p.add_argument("--train-height", type=int, default=840)
    p.add_argument("--train-steps", type=int, default=5)
    return p.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def relaunch_distributed(n: int) -> int:
    """Run this script under torch.distributed.run with n ranks (one node,
    127.0.0.1 rendezvous on a free port); returns its exit code."""
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def workload_name(args) -> str:
    """The headline workload, named identically by both arms."""
    return (f"config4: G({args.n},{args.seed}) 6-point convexes @ {args.width}x{args.height}, "
            "DEPTH scaling, RenderSettings() defaults; each rank renders a replica view")


def workload(args):
    from paper_2411_14974_b200 import synthetic
    arrays = synthetic.quantize32(synthetic.generate_scene(args.n, args.seed))
    cam = synthetic.bench_camera(args.width, args.height)
    return arrays, cam


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi sampling of SM clocks and throttle reasons during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self) -> dict:
        sm, mx, reasons = [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        try:
            for line in open(self.path):
                parts = [x.strip() for x in line.split(",")]
                if len(parts) < 7:
                    continue
                try:
                    sm.append(float(parts[0]))
                    mx.append(float(parts[1]))
                except ValueError:
                    continue
                for name, v in zip(names, parts[3:7]):
                    if v.lower() == "active":
                        reasons.add(name)
        except OSError:
            pass
        finally:
            if self.path and os.path.exists(self.path):
                os.unlink(self.path)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


# ----------------------------------------------------------------------------- CPU baseline (oracle port)
def cpu_sample(arrays, cam, budget_s: float, threads: int, with_backward: bool = True) -> dict:
    """Time the float64 oracle (C port of the reference) on a bounded sample:
    full prepare_view + bin_tiles, then a spread-out subset of tiles whose
    size is chosen from a probe so the sample takes ~budget_s.  The frame
    time is extrapolated linearly in the number of tiles."""
    import numpy as np

    import oracle
    from paper_2411_14974_b200 import synthetic
    cam_d = synthetic.camera_dict(cam)
    o_set = dict(cutoff=2e-4, floor=1e-4, tile=16, sh_degree=3, mode="depth", background=np.zeros(3))
    t0 = time.perf_counter()
    view = oracle.prepare_view(arrays, cam_d, o_set, n_threads=threads)
    t1 = time.perf_counter()
    tiles = oracle.bin_tiles(view, cam.width, cam.height, 16)
    t2 = time.perf_counter()
    T = tiles[0].size - 1
    rng = np.random.default_rng(0)
    perm = rng.permutation(T)
    probe = perm[: max(T // 256, 8)]
    tp = time.perf_counter()
    oracle.render(arrays, cam_d, o_set, n_threads=threads, view=view, tiles=tiles, tile_list=probe)
    per_tile = (time.perf_counter() - tp) / probe.size
    count = int(min(T, max(probe.size, budget_s / max(per_tile, 1e-9) / (3.0 if with_backward else 1.0))))
    sample = np.sort(perm[:count])
    t3 = time.perf_counter()
    oracle.render(arrays, cam_d, o_set, n_threads=threads, view=view, tiles=tiles, tile_list=sample)
    t4 = time.perf_counter()
    fwd_s = (t1 - t0) + (t2 - t1) + (t4 - t3) * T / count
    out = dict(prepare_s=t1 - t0, bin_s=t2 - t1, tiles_sampled=count, tiles_total=T,
               render_sample_s=t4 - t3, fwd_frame_s=fwd_s)
    if with_backward:
        d_img = np.random.default_rng(0).normal(0.0, 1e-3, size=(cam.height, cam.width, 3))
        t5 = time.perf_counter()
        oracle.backward(arrays, cam_d, o_set, d_img, n_threads=threads, view=view, tiles=tiles, tile_list=sample)
        t6 = time.perf_counter()
        # the chain over all visible convexes runs once regardless of the sample
        out.update(backward_sample_s=t6 - t5, fwd_bwd_frame_s=fwd_s + (t6 - t5) * T / count)
    return out


def run_reference(args):
    """--impl reference: the reference CPU path (oracle port) on the host cores."""
    world, rank, _ = dist_env()
    if rank != 0:
        return
    arrays, cam = workload(args)
    threads = host_cores()
    times = []
    info = None
    for i in range(args.warmup + args.steps):
        budget = max(2.0, min(args.cpu_budget_s, 120.0 / max(args.warmup + args.steps, 1)))
        info = cpu_sample(arrays, cam, budget, threads, with_backward=False)
        if i >= args.warmup:
            times.append(info["fwd_frame_s"])
    frame_s = statistics.mean(times)
    value = 1.0 / frame_s
    sample = (f"G({args.n},{args.seed}) @{args.width}x{args.height}: full prepare_view+bin_tiles, "
              f"{info['tiles_sampled']}/{info['tiles_total']} tiles rendered per step, frame time extrapolated")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": frame_s * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload_name(args),
                       "impl_detail": "oracle/cs_oracle.c float64 C port of convexsplat 0.1.0 (reference is "
                                      "pure NumPy; not compiled), OpenMP over tiles"},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port", "sample": sample,
                             "cpu": cpu_model()},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- configs 1-3
def graph_times(r, fr, d_image, grads, flush, dev, steps: int, warmup: int, backward: bool):
    """Forward (and forward + backward with fresh gradients) of an existing
    frame as CUDA-graph replays, L2 flushed before every timed step; mean ms."""
    import numpy as np
    import torch
    stream = torch.cuda.current_stream(dev)

    def capture(fn):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            fn()
        return g

    def fwdbwd():
        r.launch_forward(fr, 0, 2, zero_accumulators=True)   # the accumulator reset runs under the forward
        r.launch_backward(fr, d_image, grads, 0, 0)
        r.launch_backward(fr, d_image, grads, 1, 1, overwrite=True)

    torch.cuda.synchronize(dev)
    graphs = [capture(lambda: r.launch_forward(fr, 0, 2))] + ([capture(fwdbwd)] if backward else [])
    torch.cuda.synchronize(dev)
    out = []
    for g in graphs:
        for _ in range(warmup):
            g.replay()
        ms = []
        for _ in range(steps):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            g.replay()
            e1.record(stream)
            torch.cuda.synchronize(dev)
            ms.append(e0.elapsed_time(e1))
        out.append(float(np.mean(ms)))
    return out


def config1_block(args, dev, flush, cpu: bool) -> dict:
    """BASELINE.json configs[0]: the reference's own config-1 scene
    (synth.make_scene(1000, 6, seed=0), ring_cameras(1, size=256)[0]; the
    committed fixture tests/golden/config1.npz made by the reference) and its
    d_image; forward + backward."""
    import numpy as np
    import torch

    import paper_2411_14974_b200 as cs
    from paper_2411_14974_b200 import rasterizer as rz
    from tests import golden_cases as gc
    g = gc.load("config1")
    c, st_d = gc.camera(g), gc.settings(g)
    cam = cs.Camera(fx=c["fx"], fy=c["fy"], cx=c["cx"], cy=c["cy"], width=c["width"], height=c["height"], R=c["R"],
                    t=c["t"], z_near=c["z_near"], ortho=c["ortho"])
    settings = cs.RenderSettings(contribution_cutoff=st_d["cutoff"], transmittance_floor=st_d["floor"])
    st = cs.SceneTensors.from_arrays(gc.params(g), dev, background=g["background"])
    r = rz.Rasterizer(dev)
    fr = r.forward(st, cam, cs.ScalingMode(st_d["mode"]), settings)
    d = torch.tensor(g["d_image"], dtype=torch.float32, device=dev)
    fwd_ms, fb_ms = graph_times(r, fr, d, rz.empty_grads(st), flush, dev, max(args.steps, 20), 3, True)
    out = {"workload": "config1: reference make_scene(1000, 6, seed=0) @ ring_cameras(1, size=256)[0], its d_image "
                       "(tests/golden/config1.npz)", "convexes": st.n, "pairs": fr.n_pairs,
           "gpu": {"fwd_fps": 1000.0 / fwd_ms, "fwd_ms": fwd_ms, "fwd_bwd_iters_per_s": 1000.0 / fb_ms,
                   "fwd_bwd_ms": fb_ms, "launch": "CUDA graph replay, L2 flushed between steps"}}
    if cpu:
        import oracle
        threads = host_cores()
        t0 = time.perf_counter()
        reps = 0
        while reps < 3 or time.perf_counter() - t0 < 2.0:
            view = oracle.prepare_view(gc.params(g), c, st_d, n_threads=threads)
            tiles = oracle.bin_tiles(view, c["width"], c["height"], 16)
            oracle.render(gc.params(g), c, st_d, n_threads=threads, view=view, tiles=tiles)
            reps += 1
        t_f = (time.perf_counter() - t0) / reps
        t0 = time.perf_counter()
        oracle.backward(gc.params(g), c, st_d, g["d_image"], n_threads=threads)
        t_b = time.perf_counter() - t0
        out["cpu_baseline"] = {"kind": "port", "cores": threads, "cpu": cpu_model(),
                               "fwd_fps": 1.0 / t_f, "fwd_bwd_iters_per_s": 1.0 / (t_f + t_b),
                               "sample": "whole frame (float64 C oracle: prepare_view + bin_tiles + render; backward "
                                         "re-walks the frame)",
                               "reference_numpy_s": {"fwd": 1.07, "bwd": 3.17, "source": "BASELINE.md section 2 "
                                                     "(the reference package itself, 1 core, survey container)"}}
    return out


def config3_block(args, dev, flush, cpu: bool) -> dict:
    """BASELINE.json configs[2]: G(100k, 0) @ C(1297, 840), forward FPS."""
    import paper_2411_14974_b200 as cs
    from paper_2411_14974_b200 import rasterizer as rz, synthetic
    arrays = synthetic.quantize32(synthetic.generate_scene(100_000, 0))
    cam = synthetic.bench_camera(1297, 840)
    st = cs.SceneTensors.from_arrays(arrays, dev)
    r = rz.Rasterizer(dev)
    fr = r.forward(st, cam, cs.ScalingMode.DEPTH, cs.RenderSettings())
    (fwd_ms,) = graph_times(r, fr, None, None, flush, dev, max(args.steps, 20), 3, False)
    out = {"workload": "config3: G(100000,0) 6-point convexes @ 1297x840 (Mip-NeRF360 /4 shape), forward",
           "convexes": st.n, "pairs": fr.n_pairs,
           "gpu": {"fwd_fps": 1000.0 / fwd_ms, "fwd_ms": fwd_ms, "launch": "CUDA graph replay, L2 flushed"}}
    if cpu:
        threads = host_cores()
        c = cpu_sample(arrays, cam, 6.0, threads, with_backward=False)
        out["cpu_baseline"] = {"kind": "port", "cores": threads, "cpu": cpu_model(), "fwd_fps": 1.0 / c["fwd_frame_s"],
                               "sample": f"full prepare_view+bin_tiles + {c['tiles_sampled']}/{c['tiles_total']} "
                                         "random tiles, extrapolated",
                               "reference_numpy_s": {"fwd": 70.5, "source": "BASELINE.md section 2"}}
    return out


def config2_block(args, dev, cpu: bool) -> dict:
    """BASELINE.json configs[1]: toy chair fit.  Ground truth: the procedural
    chair of 6-point prisms (synthetic.chair_scene) rendered from
    ring_cameras(128) at 512^2; the fitted scene starts from
    initialize.init_scene semantics on 2000 surface samples
    (synthetic.init_scene_arrays).  One training step = render + L1/D-SSIM +
    mask loss + backward of all 128 views, summed gradients, fused Adam
    (ViewShardedStep, batch = 128 views)."""
    import numpy as np
    import torch

    import paper_2411_14974_b200 as cs
    from paper_2411_14974_b200 import rasterizer as rz, sharded, synthetic
    size, nv = args.chair_size, args.chair_views
    cams = synthetic.ring_cameras(nv, size, size)
    mode, settings = cs.ScalingMode.DEPTH, cs.RenderSettings()
    r = rz.Rasterizer(dev)
    gt = cs.SceneTensors.from_arrays(synthetic.quantize32(synthetic.chair_scene()), dev)
    views = [(c, r.forward(gt, c, mode, settings).image.clone()) for c in cams]
    pts, cols = synthetic.chair_surface_samples(2000, seed=0)
    init = synthetic.quantize32(synthetic.init_scene_arrays(pts, cols))
    scene = cs.SceneTensors.from_arrays(init, dev)
    params = {k: getattr(scene, k) for k in sharded.PARAM_ORDER}
    step = sharded.ViewShardedStep(params, sharded.StepConfig(),
                                   sharded.rasterizer_view_grad_fn(scene, mode, settings, rasterizer=r))
    stream = torch.cuda.current_stream(dev)
    step.step(views)                                     # warm-up: sizes the pair capacity
    torch.cuda.synchronize(dev)
    times, losses = [], []
    for _ in range(args.chair_steps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        info = step.step(views)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        times.append(e0.elapsed_time(e1))
        losses.append(float(info["local_loss_sum"]) / nv)
    ms = float(np.mean(times))
    out = {"workload": f"config2: toy chair fit, {scene.n} convexes initialised from 2000 chair surface samples "
                       f"(initialize.init_scene semantics), {nv} ring views @ {size}x{size}, batch = all views",
           "gt_convexes": gt.n, "convexes": scene.n,
           "gpu": {"train_steps_per_s": 1000.0 / ms, "ms_per_step": ms, "views_per_s": nv * 1000.0 / ms,
                   "mean_view_loss_first_last": [losses[0], losses[-1]], "steps": args.chair_steps,
                   "step": "per view: forward, fused L1+D-SSIM+mask loss, backward (accumulate); views alternate "
                           "between 4 CUDA-stream lanes; then one fused Adam update"}}
    if cpu:
        import oracle
        threads = host_cores()
        o_set = dict(cutoff=2e-4, floor=1e-4, tile=16, sh_degree=3, mode="depth", background=np.zeros(3))
        sample = 2
        t0 = time.perf_counter()
        for c, tgt in views[:sample]:
            cam_d = synthetic.camera_dict(c)
            view = oracle.prepare_view(init, cam_d, o_set, n_threads=threads)
            tiles = oracle.bin_tiles(view, size, size, 16)
            fr = oracle.render(init, cam_d, o_set, n_threads=threads, view=view, tiles=tiles)
            img = torch.tensor(fr["image"], requires_grad=True)
            raw_mask = torch.tensor(init["raw_mask"], requires_grad=True)
            loss = sharded.image_loss(img, tgt.double().cpu(), raw_mask)["total"]
            d_img, _ = torch.autograd.grad(loss, (img, raw_mask))
            oracle.backward(init, cam_d, o_set, d_img.numpy(), n_threads=threads, view=view, tiles=tiles)
        per_view = (time.perf_counter() - t0) / sample
        out["cpu_baseline"] = {"kind": "port", "cores": threads, "cpu": cpu_model(),
                               "train_steps_per_s": 1.0 / (per_view * nv),
                               "sample": f"{sample} of {nv} views (float64 C oracle fwd+bwd, torch float64 loss on "
                                         f"the CPU), extrapolated to the {nv}-view step"}
    return out


# ----------------------------------------------------------------------------- config 5
def train_step_bench(args, st, arrays, dev, world, rank):
    """One optimisation step over a batch of B ring views (1297x840): views
    sharded round-robin over the ranks, device loss (L1 + D-SSIM + mask),
    backward through the C ABI into one flat buffer, one NCCL all_reduce,
    Adam on every rank.  Targets are renders of a perturbed scene."""
    import torch
    import torch.distributed as dist

    from paper_2411_14974_b200 import sharded, synthetic
    from paper_2411_14974_b200.model import RenderSettings, ScalingMode
    from paper_2411_14974_b200.rasterizer import Rasterizer
    from paper_2411_14974_b200.scene_tensors import SceneTensors

    cams = synthetic.ring_cameras(args.train_views, args.train_width, args.train_height)
    mode, settings = ScalingMode.DEPTH, RenderSettings()
    r = Rasterizer(dev)
    tgt = SceneTensors.from_arrays(synthetic.quantize32(synthetic.perturb(arrays, seed=1)), dev)
    mine = set(sharded.shard_views(list(range(len(cams))), rank, world))
    views = [(c, r.forward(tgt, c, mode, settings).image.clone() if i in mine else None) for i, c in enumerate(cams)]
    del tgt
    scene = SceneTensors(*(getattr(st, k).clone() for k in ("points", "raw_delta", "raw_sigma", "raw_opacity",
                                                            "raw_mask", "sh")), background=st.background)
    params = {k: getattr(scene, k) for k in sharded.PARAM_ORDER}
    step = sharded.ViewShardedStep(params, sharded.StepConfig(),
                                   sharded.rasterizer_view_grad_fn(scene, mode, settings, rasterizer=r))
    stream = torch.cuda.current_stream(dev)
    step.step(views)                                   # warm-up (sizes every view's pair capacity)
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    times, losses = [], []
    for _ in range(args.train_steps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        info = step.step(views)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        times.append(e0.elapsed_time(e1))
        losses.append(float(info["local_loss_sum"]))
    t = torch.tensor([sum(times) / len(times)], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t[0])
    return {"metric": "view-sharded training steps/s (config 5)", "steps_per_s": 1000.0 / ms, "ms_per_step": ms,
            "views_per_s": args.train_views * 1000.0 / ms, "batch_views": args.train_views,
            "view_size": [args.train_width, args.train_height], "convexes": st.n, "ranks": world,
            "views_per_rank": len(mine), "steps": args.train_steps, "scaling": "strong (fixed batch of views)",
            "lanes": "views alternate between 4 CUDA-stream lanes (own workspaces) on each rank",
            "collective": "one all_reduce(SUM) of %d float32 per step" % step.flat.buffer.numel(),
            "rank0_loss_sum_first_last": [losses[0], losses[-1]]}


# ----------------------------------------------------------------------------- launcher check (CPU)
def cpu_check(args):
    """--cpu-check: the multi-rank plumbing of this script without a GPU.
    Every rank runs the config-5 step logic (ViewShardedStep: round-robin
    views, one all_reduce(SUM) per step, identical Adam) with the
    deterministic CPU per-view gradients of tests/test_sharded.py over gloo;
    rank 0 prints the world size it ran with and whether every replica ended
    bit-identical to the others and to a single-process run."""
    import torch
    import torch.distributed as dist

    from paper_2411_14974_b200 import sharded
    from tests.test_sharded import _params, _run_steps

    world, rank, _ = dist_env()
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    batch, steps = list(range(2 * world + 3)), 3
    single = _params()                    # the single-process result (before the group exists)
    _run_steps(single, batch, steps)
    if world > 1:
        dist.init_process_group("gloo")
    params = _params()
    _run_steps(params, batch, steps)
    flat = torch.cat([params[k].reshape(-1) for k in sharded.PARAM_ORDER])
    gathered = [torch.empty_like(flat) for _ in range(world)]
    if world > 1:
        dist.all_gather(gathered, flat)
    else:
        gathered = [flat]
    if rank == 0:
        ref = torch.cat([single[k].reshape(-1) for k in sharded.PARAM_ORDER])
        line = {"impl": "cpu-check", "n_gpus": world, "ranks": len(gathered), "backend": "gloo" if world > 1 else None,
                "views": len(batch), "steps": steps,
                "replicas_identical": all(torch.equal(g, gathered[0]) for g in gathered),
                "max_abs_vs_single_process": float((gathered[0] - ref).abs().max())}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


# ----------------------------------------------------------------------------- GPU arm
def main():
    args = parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch_distributed(args.gpus))     # one process per GPU under torch.distributed.run
    if args.impl == "reference":
        run_reference(args)
        return
    if args.cpu_check:
        cpu_check(args)
        return
    import numpy as np
    import torch
    import torch.distributed as dist

    world, rank, local = dist_env()
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        # communicator set-up (ranks, transports, NVLS) on stderr
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        dist.init_process_group("nccl", device_id=dev)

    from paper_2411_14974_b200 import rasterizer as rz
    from paper_2411_14974_b200.model import RenderSettings, ScalingMode
    from paper_2411_14974_b200.scene_tensors import SceneTensors

    arrays, cam = workload(args)
    st = SceneTensors.from_arrays(arrays, dev)
    r = rz.Rasterizer(dev)
    ws = rz.Workspace(dev)
    settings = RenderSettings()
    fr = r.forward(st, cam, ScalingMode.DEPTH, settings, workspace=ws)      # sizes the pair capacity
    gen = torch.Generator(device=dev).manual_seed(args.seed)
    d_image = torch.randn((cam.height, cam.width, 3), generator=gen, device=dev) * 1e-3
    grads = rz.zero_grads(st)
    # one untimed counted pass for the work statistics (roofline accounting);
    # the timed passes run the uncounted kernels
    r.launch_forward(fr, 0, 2, work_counters=True)
    r.launch_backward(fr, d_image, grads, work_counters=True)
    stats = r.read_stats(fr)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)            # > 126 MB L2
    stream = torch.cuda.current_stream(dev)

    def barrier():
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    # The C-ABI launches of a frame are captured once into CUDA graphs and
    # replayed (stream-ordered device work only: no host sync inside a
    # frame, so a graph is exactly the frame; replay removes the launch gaps
    # between the ~15 kernels and memsets).  Whole-frame graphs give the
    # headline times; per-stage graphs give the stage breakdown.
    def capture(fn):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            fn()
        return g

    def fwdbwd():
        r.launch_forward(fr, 0, 2, zero_accumulators=True)   # the accumulator reset runs under the forward
        r.launch_backward(fr, d_image, grads, 0, 0)
        r.launch_backward(fr, d_image, grads, 1, 1, overwrite=True)   # fresh gradients, no zeroing pass

    torch.cuda.synchronize(dev)
    g_fwd = capture(lambda: r.launch_forward(fr, 0, 2))
    g_fstage = [capture(lambda k=k: r.launch_forward(fr, k, k)) for k in range(3)]
    g_fb = capture(fwdbwd)
    g_b0 = capture(lambda: r.launch_backward(fr, d_image, grads, 0, 0))
    g_b1 = capture(lambda: r.launch_backward(fr, d_image, grads, 1, 1, overwrite=True))
    torch.cuda.synchronize(dev)

    def timed(graphs, k):
        evs = [[torch.cuda.Event(enable_timing=True) for _ in range(len(graphs) + 1)] for _ in range(k)]
        for i in range(k):
            flush.zero_()                          # untimed L2 flush between frames
            evs[i][0].record(stream)
            for j, g in enumerate(graphs):
                g.replay()
                evs[i][j + 1].record(stream)
        torch.cuda.synchronize(dev)
        return np.array([[e[j].elapsed_time(e[j + 1]) for j in range(len(graphs))] for e in evs])   # ms

    for _ in range(args.warmup):
        timed([g_fwd], 1)
        timed(g_fstage, 1)
        timed([g_fb], 1)
        timed([g_fwd, g_b0, g_b1], 1)
    barrier()
    with ClockSampler(local) as clocks:
        barrier()
        fwd_whole = timed([g_fwd], args.steps)
        barrier()
        fwd = timed(g_fstage, args.steps)
        barrier()
        fb_whole = timed([g_fb], args.steps)
        barrier()
        fb = timed([g_fwd, g_b0, g_b1], args.steps)
        barrier()
    clock = clocks.summary()
    fwd_ms_local = float(fwd_whole.sum(axis=1).mean())
    fb_ms_local = float(fb_whole.sum(axis=1).mean())
    t = torch.tensor([fwd_ms_local, fb_ms_local], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    fwd_ms, fb_ms = float(t[0]), float(t[1])

    # ---- e2e: host buffers through the C-ABI call.  Every frame copies its
    # full parameter set from pinned host memory and reads its image back;
    # double-buffered device parameter sets let frame i+1's H2D copy (copy
    # stream) overlap frame i's render, and the D2H of frame i runs on a third
    # stream (the other copy engine).  Time = first copy issue -> last image
    # on the host, divided by the frame count.
    e2e = None
    if not args.no_e2e:
        names = ("points", "raw_delta", "raw_sigma", "raw_opacity", "raw_mask", "sh")
        # the parameters live in ONE pinned host block (and one device block
        # per set, the fields 256-byte aligned views into it): one 280 MB copy
        # per frame instead of six, so the copy engine streams back to back
        shapes = [tuple(getattr(st, k).shape) for k in names]
        sizes = [int(np.prod(sh_)) for sh_ in shapes]
        offs, o = [], 0
        for z in sizes:
            offs.append(o)
            o += (z + 63) // 64 * 64
        host_block = torch.zeros(o, dtype=torch.float32).pin_memory()
        for k, off, z in zip(names, offs, sizes):
            host_block[off:off + z].copy_(getattr(st, k).detach().reshape(-1).cpu())

        def device_set():
            blk = host_block.to(dev)   # starts as the real parameters (the sizing forward sees them)
            views = [blk[off:off + z].view(sh_) for off, z, sh_ in zip(offs, sizes, shapes)]
            return blk, SceneTensors(*views, background=st.background)

        blocks, sets = zip(*(device_set() for _ in range(2)))
        frames = [r.forward(sets[b], cam, ScalingMode.DEPTH, settings, workspace=ws) for b in range(2)]
        img_host = [torch.empty(fr.image.shape, dtype=torch.float32).pin_memory() for _ in range(2)]
        h2d = o * 4   # bytes copied per frame (the fields plus <= 255 B of alignment each)
        d2h = img_host[0].numel() * 4
        cs_, ds_ = torch.cuda.Stream(dev), torch.cuda.Stream(dev)

        def e2e_run(k):
            copied = [torch.cuda.Event() for _ in range(k)]
            rendered = [torch.cuda.Event() for _ in range(k)]
            fetched = [torch.cuda.Event() for _ in range(k)]
            start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            start.record(stream)
            cs_.wait_event(start)
            for i in range(k):
                b = i % 2
                with torch.cuda.stream(cs_):
                    if i >= 2:
                        cs_.wait_event(rendered[i - 2])          # set b free again
                    blocks[b].copy_(host_block, non_blocking=True)
                    copied[i].record(cs_)
                stream.wait_event(copied[i])
                if i >= 2:
                    stream.wait_event(fetched[i - 2])            # image buffer b read back
                r.launch_forward(frames[b], 0, 2)
                rendered[i].record(stream)
                with torch.cuda.stream(ds_):
                    ds_.wait_event(rendered[i])
                    img_host[b].copy_(frames[b].image, non_blocking=True)
                    fetched[i].record(ds_)
            stream.wait_event(fetched[k - 1])
            end.record(stream)
            torch.cuda.synchronize(dev)
            return start.elapsed_time(end) / k

        e2e_run(max(args.warmup, 2))
        barrier()
        e2e_local = e2e_run(args.steps)
        te = torch.tensor([e2e_local], device=dev, dtype=torch.float64)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e = {"value": world * 1000.0 / float(te[0]), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "ms_per_step": float(te[0]),
               "path": "pinned host params (one block) -> cs_forward (C ABI) -> pinned host image; two device "
                       "parameter sets: H2D of frame i+1 overlaps the render of frame i, D2H on a third stream"}

    # ---- roofline: SURVEY.md 8(d)'s algorithmic work per stage
    L = ws.layout
    n, V, P = st.n, stats["n_visible"], stats["n_pairs"]
    pp = max(1, math.ceil(math.log2(max(L.tiles_x * L.tiles_y, 2)) / 8))
    stage_ms = fwd.mean(axis=0)
    bwd_ms = fb.mean(axis=0)
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except (OSError, ValueError):
        pass
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    sm_max = float(peaks.get("sm_max_mhz", 1965.0))
    mufu_peak = N_SMS * MUFU_PER_CLK_PER_SM * sm_max * 1e6 / 1e9          # Gop/s, derived
    mufu_source = (f"derived: {N_SMS} SMs x {MUFU_PER_CLK_PER_SM} MUFU/clk x {sm_max:.0f} MHz "
                   "(sm_max_mhz of MEASURED_PEAKS.json)")
    try:   # measured on a B200 by tools/mufu_peak.cu (ex2 throughput at the max SM clock)
        mp = json.load(open(os.path.join(ROOT, "profiles", "mufu_peak.json")))
        mufu_peak = float(mp["mufu_ex2_gops"]) * sm_max / float(mp["sm_clock_mhz"])
        mufu_source = (f"measured: tools/mufu_peak.cu, {mp['mufu_ex2_gops']} Gop/s ex2 at {mp['sm_clock_mhz']} MHz "
                       f"({mp['per_sm_per_clk']} per SM per clock; profiles/mufu_peak.json)")
    except (OSError, ValueError, KeyError):
        pass
    # K1: params read (280 B) + tiles_touched (4 B) per convex, 104-B record per visible convex
    pre_bytes = n * 280 + n * 4 + V * 104
    # K2: depth rank V x 12 B x 2 x 8 passes; duplicate P x 12 B; radix over
    # ceil(log2 tiles) + ceil(log2 V) key bits in 8-bit digits, P x (2 x 12 x passes + 8) B; ranges P x 8 B
    key_bits = math.ceil(math.log2(max(L.tiles_x * L.tiles_y, 2))) + math.ceil(math.log2(max(V, 2)))
    radix_passes = math.ceil(key_bits / 8)
    bin_bytes = V * 12 * 2 * 8 + P * 12 + P * (2 * 12 * radix_passes + 8) + P * 8
    # K3: E_fwd x (T + 2) MUFU ops (T = hull lines of the candidate; E_fwd from the counting run)
    fwd_mufu = stats["fwd_line_evals"] + 2 * stats["fwd_evals"]
    # K4a: E_bwd x (T + 3); K4b: N x (280 + 96 + 280) B
    bwd_mufu = stats["bwd_line_evals"] + 3 * stats["bwd_evals"]
    chain_bytes = n * (280 + 96 + 280)

    def stage(ms, bound, work, unit, peak, basis):
        achieved = work / (ms * 1e-3) / 1e9
        return {"ms": float(ms), "bound": bound, "work": int(work), "unit": unit, "achieved": achieved,
                "peak": peak, "frac": achieved / peak, "ideal_ms": work / peak / 1e9 * 1e3, "basis": basis}
    stage_info = {
        "preprocess": stage(stage_ms[0], "hbm", pre_bytes, "GB/s", hbm_peak, "N x 284 B + V x 104 B"),
        "binning": stage(stage_ms[1], "hbm", bin_bytes, "GB/s", hbm_peak,
                         f"V x 192 B + P x (12 + 24 x {radix_passes} + 16) B ({key_bits}-bit keys)"),
        "blend": stage(stage_ms[2], "sfu", fwd_mufu, "Gop/s", mufu_peak, "E_fwd x (T + 2) MUFU"),
        "backward_blend": stage(bwd_ms[1], "sfu", bwd_mufu, "Gop/s", mufu_peak, "E_bwd x (T + 3) MUFU"),
        "chain": stage(bwd_ms[2], "hbm", chain_bytes, "GB/s", hbm_peak, "N x (280 + 96 + 280) B"),
    }
    ideal_fwd = sum(stage_info[k]["ideal_ms"] for k in ("preprocess", "binning", "blend"))
    ideal_fb = ideal_fwd + stage_info["backward_blend"]["ideal_ms"] + stage_info["chain"]["ideal_ms"]
    composite = {"forward": {"ideal_ms": ideal_fwd, "measured_ms": fwd_ms, "frac": ideal_fwd / fwd_ms},
                 "fwd_bwd": {"ideal_ms": ideal_fb, "measured_ms": fb_ms, "frac": ideal_fb / fb_ms}}
    dominant = max(stage_info, key=lambda s2: stage_info[s2]["ms"])      # over the fwd+bwd frame
    dom = stage_info[dominant]
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(prof):
        try:
            traffic = json.load(open(prof)).get(dominant)
        except ValueError:
            traffic = None
    roofline = {"kernel": dominant, "bound": dom["bound"], "achieved": dom["achieved"], "peak": dom["peak"],
                "unit": dom["unit"], "frac": dom["frac"], "traffic": traffic,
                "peak_source": "MEASURED_PEAKS.json hbm_gbs" if dom["bound"] == "hbm" else mufu_source,
                "work_source": "SURVEY.md 8(d) algorithmic counts; E and T from an untimed counting pass",
                "stages": stage_info, "composite": composite}

    configs = None
    if world == 1 and not args.no_configs:
        del fr, grads
        torch.cuda.empty_cache()
        cpu_ok = not args.no_cpu_baseline
        configs = {"config1": config1_block(args, dev, flush, cpu_ok),
                   "config3": config3_block(args, dev, flush, cpu_ok),
                   "config2": config2_block(args, dev, cpu_ok)}
        torch.cuda.empty_cache()

    # ---- config 5: view-sharded training step (B views, all_reduce of the gradients)
    train = None
    if not args.no_train:
        train = train_step_bench(args, st, arrays, dev, world, rank)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = host_cores()
        cs_ = cpu_sample(arrays, cam, args.cpu_budget_s, threads, with_backward=True)
        cpu = {"value": 1.0 / cs_["fwd_frame_s"], "unit": UNIT, "cores": threads, "kind": "port",
               "sample": (f"float64 C oracle (oracle/cs_oracle.c), full prepare_view+bin_tiles of G({args.n}) "
                          f"+ {cs_['tiles_sampled']}/{cs_['tiles_total']} random tiles, extrapolated"),
               "fwd_bwd_iters_per_s": 1.0 / cs_["fwd_bwd_frame_s"], "cpu": cpu_model(), "detail": cs_}

    launches_fwd = 13 + pp
    line = {
        "metric": METRIC, "value": world * 1000.0 / fwd_ms, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": fwd_ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32 (f64 preprocess)", "data": "synthetic",
        "config": {"workload": workload_name(args),
                   "convexes": n, "width": args.width, "height": args.height, "visible": V, "pairs": P,
                   "l2": "flushed before every timed step (512 MB write, untimed)",
                   "launch": "CUDA graph replay of the frame's C-ABI launches (captured once)",
                   "parallelism": f"replicas x{world}"},
        "fwd_bwd_iters_per_s": world * 1000.0 / fb_ms, "fwd_bwd_ms": fb_ms,
        "stage_ms": {"preprocess": float(stage_ms[0]), "binning": float(stage_ms[1]), "blend": float(stage_ms[2]),
                     "fwd_total": float(fwd.sum(axis=1).mean()), "forward(fwd+bwd)": float(bwd_ms[0]),
                     "backward_blend": float(bwd_ms[1]), "chain": float(bwd_ms[2])},
        "work": {k2: int(v) for k2, v in stats.items()},
        "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "clocks": clock, "train_step": train,
        "configs": configs,
        # timed: whole-frame and per-stage graphs of the forward, then of fwd+bwd
        "gpu_launches": 2 * args.steps * (launches_fwd + (launches_fwd + 3)),
        "gpu_launches_detail": f"{launches_fwd} per forward (1 preprocess, 1 scratch clear, 6 depth order: key32 + offsets + "
                               f"3 onesweep + fix-up, 1 scan+duplicate, {1 + pp} pair sort, 1 ranges, 1 tile order, "
                               f"1 blend), 3 per backward (accumulator zeroing, blend, chain); each timed "
                               f"twice (whole-frame graph, per-stage graphs)",
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
