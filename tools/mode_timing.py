"""Forward / fwd+bwd time per scaling mode at 1M @1080p (CUDA events, graphs not used)."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2411_14974_b200 as cs
from paper_2411_14974_b200 import rasterizer as rz, synthetic

arrays = synthetic.quantize32(synthetic.generate_scene(1_000_000, 0))
cam = synthetic.bench_camera(1920, 1080)
st = cs.SceneTensors.from_arrays(arrays, "cuda")
r = rz.Rasterizer("cuda")
d = torch.randn(1080, 1920, 3, device="cuda") * 1e-3
for name, mode in (("depth", cs.ScalingMode.DEPTH), ("sqrt", cs.ScalingMode.SQRT_DEPTH),
                   ("none", cs.ScalingMode.NONE), ("depth2", cs.ScalingMode.DEPTH_SQUARED)):
    fr = r.forward(st, cam, mode, cs.RenderSettings())
    g = rz.zero_grads(st)
    for _ in range(3):
        r.launch_forward(fr, 0, 2)
        r.launch_backward(fr, d, g, overwrite=True)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    ts = []
    for _ in range(10):
        ev[0].record(); r.launch_forward(fr, 0, 2); ev[1].record(); r.launch_backward(fr, d, g, overwrite=True); ev[2].record()
        torch.cuda.synchronize()
        ts.append((ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2])))
    f = sorted(t[0] for t in ts)[5]; b = sorted(t[1] for t in ts)[5]
    print(f"{name:7s} forward {f:.3f} ms  backward {b:.3f} ms  pairs {fr.n_pairs}")
