"""Config 2 (toy chair fit, BASELINE.json configs[1]) on the GPU: one
training step's summed gradients against the float64 oracle.

The step's flat gradient buffer (ViewShardedStep.accumulate: per view the
sm_100a render, the fused L1 + D-SSIM + mask loss, the backward accumulating
into the buffer) equals the sum over views of the float64 oracle backward of
each view's d_image at the GPU's blend decisions, plus the mask-loss term
beta * sigmoid'(raw_mask) / n per view (losses.py:151-155, trainer.py:176)."""
import numpy as np
import pytest
import torch

import oracle
from tests.test_gpu_parity import check_grads_forced

pytestmark = pytest.mark.gpu


def test_chair_step_gradients_match_oracle():
    import paper_2411_14974_b200 as cs
    from paper_2411_14974_b200 import rasterizer as rz, sharded, synthetic
    from paper_2411_14974_b200.train_ops import image_loss
    size, nv = 96, 3
    cams = synthetic.ring_cameras(nv, size, size)
    mode, settings = cs.ScalingMode.DEPTH, cs.RenderSettings()
    r = rz.Rasterizer("cuda")
    gt = cs.SceneTensors.from_arrays(synthetic.quantize32(synthetic.chair_scene()), "cuda")
    views = [(c, r.forward(gt, c, mode, settings).image.clone()) for c in cams]
    pts, cols = synthetic.chair_surface_samples(300, seed=1)
    init = synthetic.quantize32(synthetic.init_scene_arrays(pts, cols))
    scene = cs.SceneTensors.from_arrays(init, "cuda")
    params = {k: getattr(scene, k) for k in sharded.PARAM_ORDER}
    cfg = sharded.StepConfig()
    step = sharded.ViewShardedStep(params, cfg, sharded.rasterizer_view_grad_fn(scene, mode, settings, config=cfg))
    step.accumulate(views)
    gpu = {k: step.flat.views[k].detach().cpu().numpy() for k in sharded.PARAM_ORDER}
    n = scene.n
    o_set = dict(cutoff=2e-4, floor=1e-4, tile=16, sh_degree=3, mode="depth", background=np.zeros(3))
    total = {k: 0.0 for k in ("d_points", "d_raw_delta", "d_raw_sigma", "d_raw_opacity", "d_sh", "d_raw_mask")}
    m = 1.0 / (1.0 + np.exp(-init["raw_mask"]))
    for cam, target in views:
        fr = r.forward(scene, cam, mode, settings)
        loss = image_loss(fr.image, target, scene.raw_mask, cfg.lambda_dssim, cfg.beta_mask,
                          d_raw_mask=torch.zeros_like(scene.raw_mask))
        d_img = loss["d_image"].double().cpu().numpy()
        forced = rz.record_blends(fr)
        cam_d = synthetic.camera_dict(cam)
        og = oracle.backward(init, cam_d, o_set, d_img, n_threads=8, forced=forced)
        for k in total:
            total[k] = total[k] + og[k]
        total["d_raw_mask"] = total["d_raw_mask"] + cfg.beta_mask * m * (1.0 - m) / n
    check_grads_forced(gpu, total, n, f"chair step ({nv} views @{size}^2, {n} convexes)")
