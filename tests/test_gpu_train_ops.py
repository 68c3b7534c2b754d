"""GPU parity of the training-step kernels (cs_image_loss, cs_adam_step,
cs_backward_signal) against the reference fixtures (tests/golden/loss.npz,
made by running convexsplat.losses / optim) and the torch formulations."""
import os

import numpy as np
import pytest
import torch

from paper_2411_14974_b200 import sharded
from tests import golden_cases as gc

pytestmark = pytest.mark.gpu


def _ops():
    from paper_2411_14974_b200 import train_ops
    return train_ops


def test_cuda_image_loss_matches_reference_fixture():
    """losses.image_loss known answers (losses.py:129-155) on a 23x31 image."""
    ops = _ops()
    g = np.load(os.path.join(gc.GOLDEN, "loss.npz"))
    img = torch.tensor(g["img"], dtype=torch.float32, device="cuda")
    target = torch.tensor(g["target"], dtype=torch.float32, device="cuda")
    masks = torch.tensor(g["masks"], dtype=torch.float32, device="cuda")
    d_mask = torch.zeros_like(masks)
    out = ops.image_loss(img, target, masks, 0.2, 0.0005, d_raw_mask=d_mask)
    # inputs were rounded to float32: compare against the float64 reference at float32 accuracy
    assert abs(float(out["total"]) - float(g["total"])) < 2e-6
    assert abs(float(out["l1"]) - float(g["l1"])) < 1e-6
    assert abs(float(out["dssim"]) - float(g["dssim"])) < 2e-6
    assert abs(float(out["mask_term"]) - float(g["mask_term"])) < 1e-6
    d = out["d_image"].cpu().numpy()
    scale = np.abs(g["d_image"]).max()
    assert np.abs(d - g["d_image"]).max() < 1e-4 * scale
    np.testing.assert_allclose(d_mask.cpu().numpy(), g["d_raw_mask"], rtol=1e-5, atol=1e-12)


@pytest.mark.parametrize("h,w,seed", [(11, 11, 0), (70, 100, 1), (257, 130, 2)])
def test_cuda_image_loss_matches_float64_torch(h, w, seed):
    """Value and d_image vs autograd of the losses.py expression in float64
    (ragged sizes exercise the tile edges; 11x11 is the minimum image)."""
    ops = _ops()
    gen = torch.Generator().manual_seed(seed)
    img64 = torch.rand(h, w, 3, generator=gen, dtype=torch.float64)
    tgt64 = (img64 + 0.1 * torch.randn(h, w, 3, generator=gen, dtype=torch.float64)).clamp(0, 1)
    masks64 = torch.randn(50, generator=gen, dtype=torch.float64)
    img32, tgt32, m32 = (t.float().cuda() for t in (img64, tgt64, masks64))
    # reference on the float32-rounded inputs
    ri = img32.double().cpu().requires_grad_(True)
    rm = m32.double().cpu().requires_grad_(True)
    ref = sharded.image_loss(ri, tgt32.double().cpu(), rm, 0.2, 0.0005)
    d_ref, dm_ref = torch.autograd.grad(ref["total"], (ri, rm))
    dm = torch.zeros_like(m32)
    out = ops.image_loss(img32, tgt32, m32, 0.2, 0.0005, d_raw_mask=dm)
    for k in ("total", "l1", "dssim", "mask_term"):
        assert abs(float(out[k]) - float(ref[k])) < 2e-6, k
    d = out["d_image"].double().cpu()
    assert (d - d_ref).abs().max() < 1e-4 * d_ref.abs().max()
    torch.testing.assert_close(dm.double().cpu(), dm_ref, rtol=1e-5, atol=1e-12)


def test_cuda_image_loss_rejects_small_images():
    ops = _ops()
    x = torch.zeros(10, 40, 3, device="cuda")
    with pytest.raises(ValueError):
        ops.image_loss(x, x, torch.zeros(3, device="cuda"))


def test_fused_adam_matches_reference_fixture():
    """optim.Adam two steps (optim.py:22-35) from the reference fixture."""
    ops = _ops()
    g = np.load(os.path.join(gc.GOLDEN, "loss.npz"))
    params = {"a": torch.tensor(g["adam_a0"], dtype=torch.float32, device="cuda"),
              "b": torch.tensor(g["adam_b0"], dtype=torch.float32, device="cuda")}
    adam = ops.FusedAdam(params)
    for ga, gb in (("adam_ga1", "adam_gb1"), ("adam_ga2", "adam_gb2")):
        adam.step(params, {"a": torch.tensor(g[ga], dtype=torch.float32, device="cuda"),
                           "b": torch.tensor(g[gb], dtype=torch.float32, device="cuda")}, {"a": 0.01, "b": 0.002})
    np.testing.assert_allclose(params["a"].cpu().numpy(), g["adam_a2"], rtol=0, atol=2e-7)
    np.testing.assert_allclose(params["b"].cpu().numpy(), g["adam_b2"], rtol=0, atol=2e-7)


def test_fused_adam_grad_scale_and_first_step_sign():
    ops = _ops()
    p = {"x": torch.tensor([1.0, -2.0, 3.0], device="cuda"), "y": torch.zeros(5, 3, device="cuda")}
    adam = ops.FusedAdam(p)
    adam.step(p, {"x": torch.tensor([0.5, -3.0, 0.0], device="cuda"), "y": torch.ones(5, 3, device="cuda")},
              {"x": 0.1, "y": 0.5}, grad_scale=0.25)
    np.testing.assert_allclose(p["x"].cpu().numpy(), [0.9, -1.9, 3.0], atol=1e-6)   # first step = -lr sign(g)
    np.testing.assert_allclose(p["y"].cpu().numpy(), -0.5 * np.ones((5, 3)), atol=1e-6)
    idx = torch.tensor([2, -1, 0], device="cuda")
    adam.remap(idx)
    assert adam.m["x"].shape == (3,) and float(adam.m["x"][1]) == 0.0
    assert float(adam.m["x"][2]) == pytest.approx(0.1 * 0.5 * 0.25, rel=1e-6)


def test_view_signal_and_cuda_loss_step_match_torch_path():
    """ViewShardedStep.accumulate with the fused CUDA loss + in-kernel sigma
    signal equals the torch-loss path (autograd d_image, signal from the
    gradient difference): gradients within 1e-3 relative, view counts exact."""
    import paper_2411_14974_b200 as cs
    from paper_2411_14974_b200 import synthetic
    arrays = synthetic.quantize32(synthetic.generate_scene(3000, seed=4))
    st = cs.SceneTensors.from_arrays(arrays, "cuda")
    tgt = cs.SceneTensors.from_arrays(synthetic.quantize32(synthetic.perturb(arrays, seed=6)), "cuda")
    cams = synthetic.ring_cameras(4, 96, 72)
    views = [(c, torch.tensor(cs.render(tgt, c).image, dtype=torch.float32, device="cuda")) for c in cams]
    params = {k: getattr(st, k) for k in sharded.PARAM_ORDER}
    mode, settings = cs.ScalingMode.DEPTH, cs.RenderSettings()
    a = sharded.ViewShardedStep(params, sharded.StepConfig(), sharded.rasterizer_view_grad_fn(st, mode, settings))
    b = sharded.ViewShardedStep(params, sharded.StepConfig(), sharded.torch_view_grad_fn(st, mode, settings))
    a.accumulate(views)
    b.accumulate(views)
    for k in list(sharded.PARAM_ORDER) + ["sigma_signal"]:
        x, y = a.flat.views[k].cpu().numpy().ravel(), b.flat.views[k].cpu().numpy().ravel()
        den = np.maximum(np.abs(x), np.abs(y))
        rel = np.abs(x - y) / np.maximum(den, max(2e-4 * den.max(), 1e-12))
        assert rel.max() < 1e-3, (k, rel.max())
    assert torch.equal(a.flat.views["sigma_views"], b.flat.views["sigma_views"])
    assert float(a.flat.views["sigma_views"].sum()) > 0
