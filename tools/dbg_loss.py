import sys; sys.path.insert(0, ".")
import numpy as np, torch
import paper_2411_14974_b200 as cs
from paper_2411_14974_b200 import synthetic, sharded, train_ops
from paper_2411_14974_b200.rasterizer import default_rasterizer, zero_grads
arrays = synthetic.quantize32(synthetic.generate_scene(3000, seed=4))
st = cs.SceneTensors.from_arrays(arrays, "cuda")
tgt = cs.SceneTensors.from_arrays(synthetic.quantize32(synthetic.perturb(arrays, seed=6)), "cuda")
cams = synthetic.ring_cameras(4, 96, 72)
views = [(c, torch.tensor(cs.render(tgt, c).image, dtype=torch.float32, device="cuda")) for c in cams]
params = {k: getattr(st, k) for k in sharded.PARAM_ORDER}
r = default_rasterizer()
for nv in (1, 2, 4):
    a = sharded.ViewShardedStep(params, sharded.StepConfig(), sharded.rasterizer_view_grad_fn(st, cs.ScalingMode.DEPTH, cs.RenderSettings()))
    a.accumulate(views[:nv])
    ref = zero_grads(st)
    for cam, target in views[:nv]:
        fr = r.forward(st, cam)
        out = train_ops.image_loss(fr.image, target, st.raw_mask, d_raw_mask=ref["raw_mask"])
        r.launch_backward(fr, out["d_image"], ref)
    for k in ("points", "raw_delta", "sh"):
        x, y = a.flat.views[k].cpu().numpy().ravel(), ref[k].cpu().numpy().ravel()
        print(nv, k, np.abs(x - y).max(), np.abs(y).max())
