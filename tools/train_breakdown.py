"""Where the config-5 training step's time goes: per view, device time of
forward / loss / backward (CUDA events) against the host time of issuing
them.  usage: python tools/train_breakdown.py [views] [n]"""
import sys
import time

import torch

from paper_2411_14974_b200 import sharded, synthetic
from paper_2411_14974_b200.model import RenderSettings, ScalingMode
from paper_2411_14974_b200.rasterizer import Rasterizer, Workspace
from paper_2411_14974_b200.scene_tensors import SceneTensors
from paper_2411_14974_b200.train_ops import LossWorkspace, image_loss

views_n = int(sys.argv[1]) if len(sys.argv) > 1 else 8
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1_000_000
dev = torch.device("cuda")
arrays = synthetic.quantize32(synthetic.generate_scene(n, 0))
st = SceneTensors.from_arrays(arrays, dev)
tgt = SceneTensors.from_arrays(synthetic.quantize32(synthetic.perturb(arrays, seed=1)), dev)
cams = synthetic.ring_cameras(views_n, 1297, 840)
mode, settings = ScalingMode.DEPTH, RenderSettings()
r = Rasterizer(dev)
views = [(c, r.forward(tgt, c, mode, settings).image.clone()) for c in cams]
params = {k: getattr(st, k) for k in sharded.PARAM_ORDER}
step = sharded.ViewShardedStep(params, sharded.StepConfig(), sharded.rasterizer_view_grad_fn(st, mode, settings, rasterizer=r))
step.step(views)
torch.cuda.synchronize()
for _ in range(2):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    step.step(views)
    e1.record()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    print(f"step: device {e0.elapsed_time(e1):.2f} ms, host issue {1e3 * (t1 - t0):.2f} ms for {views_n} views")
# per-view stages, device side
ws, lw = Workspace(dev), LossWorkspace()
grads = {k: torch.zeros_like(v) for k, v in params.items()}
sig = torch.zeros(n, device=dev), torch.zeros(n, device=dev)
cap = None
acc = {"forward": 0.0, "loss": 0.0, "backward": 0.0}
host = 0.0
for it in range(2):
    for cam, target in views:
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        h0 = time.perf_counter()
        ev[0].record()
        fr = r.forward(st, cam, mode, settings, workspace=ws, capacity=cap, check=cap is None)
        cap = fr.capacity
        ev[1].record()
        loss = image_loss(fr.image, target, st.raw_mask, 0.2, 0.0005, d_raw_mask=grads["raw_mask"], workspace=lw)
        ev[2].record()
        r.launch_backward(fr, loss["d_image"], grads, signal=(sig[0], sig[1], fr.visible))
        ev[3].record()
        host += time.perf_counter() - h0
        torch.cuda.synchronize()
        if it == 1:
            for j, k in enumerate(acc):
                acc[k] += ev[j].elapsed_time(ev[j + 1])
print({k: round(v / views_n, 3) for k, v in acc.items()}, "ms per view (device, synchronised per view)")
print(f"host issue per view {1e3 * host / (2 * views_n):.3f} ms")
# stage split of one ring view's forward / backward (counted pass for the work numbers)
cam, target = views[0]
fr = r.forward(st, cam, mode, settings, workspace=ws)
r.launch_forward(fr, 0, 2, work_counters=True)
print("work", r.read_stats(fr))
ev = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
d_img = torch.randn_like(fr.image) * 1e-3
for _ in range(3):
    ev[0].record(); r.launch_forward(fr, 0, 0); ev[1].record(); r.launch_forward(fr, 1, 1); ev[2].record()
    r.launch_forward(fr, 2, 2); ev[3].record(); r.launch_backward(fr, d_img, grads, 0, 0); ev[4].record()
    r.launch_backward(fr, d_img, grads, 1, 1, signal=None); ev[5].record()
    torch.cuda.synchronize()
print("stages ms", [round(ev[j].elapsed_time(ev[j + 1]), 3) for j in range(5)], "(preprocess, binning, blend, bwd blend, chain)")
