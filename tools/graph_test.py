"""Forward with and without CUDA-graph replay (1M @1080p): launch gaps."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2411_14974_b200 import synthetic
from paper_2411_14974_b200 import rasterizer as rz
from paper_2411_14974_b200.model import RenderSettings, ScalingMode
from paper_2411_14974_b200.scene_tensors import SceneTensors

dev = torch.device("cuda")
arrays = synthetic.quantize32(synthetic.generate_scene(1_000_000, 0))
cam = synthetic.bench_camera(1920, 1080)
st = SceneTensors.from_arrays(arrays, dev)
r = rz.Rasterizer(dev)
fr = r.forward(st, cam, ScalingMode.DEPTH, RenderSettings(), workspace=rz.Workspace(dev))
flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    for _ in range(3):
        r.launch_forward(fr, 0, 2)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        r.launch_forward(fr, 0, 2)
    torch.cuda.synchronize()
    for mode in ("direct", "graph", "direct", "graph"):
        ts = []
        for _ in range(20):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            if mode == "graph":
                g.replay()
            else:
                r.launch_forward(fr, 0, 2)
            e1.record(s)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ts.sort()
        print(mode, f"median {ts[10] * 1000:.1f} us  min {ts[0] * 1000:.1f} us")
