"""View-sharded training step: loss / optimiser parity with the reference
(fixtures from tests/golden/make_golden.py gen_loss) and the world-size-2
sharding + all-reduce logic on CPU with the gloo backend."""
import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2411_14974_b200 import sharded
from tests import golden_cases as gc


def test_image_loss_matches_reference():
    g = np.load(os.path.join(gc.GOLDEN, "loss.npz"))
    img = torch.tensor(g["img"], dtype=torch.float64, requires_grad=True)
    target = torch.tensor(g["target"], dtype=torch.float64)
    masks = torch.tensor(g["masks"], dtype=torch.float64, requires_grad=True)
    loss = sharded.image_loss(img, target, masks, 0.2, 0.0005)
    assert abs(float(loss["total"].detach()) - float(g["total"])) < 1e-12
    assert abs(float(loss["l1"]) - float(g["l1"])) < 1e-12
    assert abs(float(loss["dssim"]) - float(g["dssim"])) < 1e-12
    assert abs(float(loss["mask_term"]) - float(g["mask_term"])) < 1e-12
    d_img, d_mask = torch.autograd.grad(loss["total"], (img, masks))
    np.testing.assert_allclose(d_img.numpy(), g["d_image"], rtol=1e-9, atol=1e-13)
    np.testing.assert_allclose(d_mask.numpy(), g["d_raw_mask"], rtol=1e-9, atol=1e-15)


def test_adam_and_position_lr_match_reference():
    g = np.load(os.path.join(gc.GOLDEN, "loss.npz"))
    params = {"a": torch.tensor(g["adam_a0"]), "b": torch.tensor(g["adam_b0"])}
    adam = sharded.Adam(params)
    adam.step(params, {"a": torch.tensor(g["adam_ga1"]), "b": torch.tensor(g["adam_gb1"])}, {"a": 0.01, "b": 0.002})
    adam.step(params, {"a": torch.tensor(g["adam_ga2"]), "b": torch.tensor(g["adam_gb2"])}, {"a": 0.01, "b": 0.002})
    np.testing.assert_allclose(params["a"].numpy(), g["adam_a2"], rtol=0, atol=1e-14)
    np.testing.assert_allclose(params["b"].numpy(), g["adam_b2"], rtol=0, atol=1e-14)
    got = [sharded.position_lr(i, 5e-4, 5e-6, 1000) for i in (0, 250, 500, 1000, 2000)]
    np.testing.assert_allclose(got, g["plr"], rtol=1e-15)


def test_adam_first_step_is_minus_lr_sign():
    p = {"x": torch.tensor([1.0, -2.0, 3.0], dtype=torch.float64)}
    adam = sharded.Adam(p)
    adam.step(p, {"x": torch.tensor([0.5, -3.0, 0.0], dtype=torch.float64)}, {"x": 0.1})
    np.testing.assert_allclose(p["x"].numpy(), [0.9, -1.9, 3.0], atol=1e-12)


def test_round_robin_sharding_covers_batch_once():
    batch = list(range(13))
    parts = [sharded.shard_views(batch, r, 4) for r in range(4)]
    assert sorted(v for part in parts for v in part) == batch
    assert parts[1] == [1, 5, 9]


def _params(seed=0, n=37, k=6):
    gen = torch.Generator().manual_seed(seed)
    f64 = dict(generator=gen, dtype=torch.float64)
    return {"points": torch.randn(n, k, 3, **f64), "raw_delta": torch.randn(n, **f64),
            "raw_sigma": torch.randn(n, **f64), "raw_opacity": torch.randn(n, **f64),
            "sh": torch.randn(n, 16, 3, **f64), "raw_mask": torch.randn(n, **f64)}


def _mock_view_grad_fn(params):
    """Deterministic per-view gradients that depend on the current parameters
    (stands in for render + loss + backward, which need the GPU)."""
    def fn(view, grads):
        v = float(view)
        for name, g in grads.items():
            g.add_(torch.sin(params[name] * (1.0 + 0.1 * v) + v))
        n = params["points"].shape[0]
        visible = (torch.arange(n) % (int(view) + 2)) != 0
        return torch.tensor(v), visible
    return fn


def _run_steps(params, batch, steps):
    step = sharded.ViewShardedStep(params, sharded.StepConfig(total_iterations=100),
                                   _mock_view_grad_fn(params))
    for _ in range(steps):
        step.step(batch)
    return step


def _worker(rank, world, port, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        params = _params()
        step = _run_steps(params, list(range(6)), 3)
        torch.save({"params": params, "sigma": step.flat.views["sigma_signal"].clone(),
                    "views": step.flat.views["sigma_views"].clone()}, f"{out_path}.{rank}")
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_two_rank_gloo_step_equals_single_process():
    """North_star 5 semantics on CPU: the 2-rank sharded step (one all_reduce
    per step) leaves both replicas identical and equal to one process
    summing all six views."""
    with tempfile.TemporaryDirectory() as tmp:
        out = os.path.join(tmp, "res")
        mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
        r0, r1 = torch.load(f"{out}.0"), torch.load(f"{out}.1")
    single_params = _params()
    single = _run_steps(single_params, list(range(6)), 3)
    for name in single_params:
        torch.testing.assert_close(r0["params"][name], r1["params"][name], rtol=0, atol=0)
        torch.testing.assert_close(r0["params"][name], single_params[name], rtol=1e-10, atol=1e-12)
    torch.testing.assert_close(r0["sigma"], single.flat.views["sigma_signal"], rtol=1e-10, atol=1e-12)
    torch.testing.assert_close(r0["views"], single.flat.views["sigma_views"], rtol=0, atol=0)


@pytest.mark.gpu
def test_sharded_step_gradients_equal_sum_of_view_backwards():
    """World size 1 on the GPU: the flat buffer after accumulate() equals the
    sum over views of rasterize-autograd gradients of the same loss."""
    import paper_2411_14974_b200 as cs
    from paper_2411_14974_b200 import synthetic
    arrays = synthetic.quantize32(synthetic.generate_scene(3000, seed=3))
    cams = synthetic.ring_cameras(3, 96, 72)
    st = cs.SceneTensors.from_arrays(arrays, "cuda")
    target_arrays = synthetic.quantize32(synthetic.perturb(arrays, seed=5))
    tgt = cs.SceneTensors.from_arrays(target_arrays, "cuda")
    views = [(c, cs.render(tgt, c).image) for c in cams]
    views = [(c, torch.tensor(t, dtype=torch.float32, device="cuda")) for c, t in views]
    params = {k: getattr(st, k) for k in sharded.PARAM_ORDER}
    mode, settings = cs.ScalingMode.DEPTH, cs.RenderSettings()
    step = sharded.ViewShardedStep(params, sharded.StepConfig(), sharded.rasterizer_view_grad_fn(st, mode, settings))
    step.accumulate(views)
    ref = {k: torch.zeros_like(v) for k, v in params.items()}
    for cam, target in views:
        leaves = {k: v.detach().clone().requires_grad_(True) for k, v in params.items()}
        scene = cs.SceneTensors(**{k: leaves[k] for k in ("points", "raw_delta", "raw_sigma", "raw_opacity",
                                                          "raw_mask", "sh")}, background=st.background)
        img = cs.rasterize(scene, cam, mode, settings)[0]
        loss = sharded.image_loss(img.double(), target.double(), leaves["raw_mask"].double())["total"]
        loss.backward()
        for k in ref:
            ref[k] += leaves[k].grad
    for k in ref:
        a, b = step.flat.views[k].cpu().numpy().ravel(), ref[k].cpu().numpy().ravel()
        den = np.maximum(np.abs(a), np.abs(b))
        # the fused loss adjoint is float32 (the reference formulation here
        # float64): the floor of tests/test_gpu_parity.py GRAD_FLOOR
        rel = np.abs(a - b) / np.maximum(den, max(5e-4 * den.max(), 1e-12))
        assert rel.max() < 1e-3, (k, rel.max())


@pytest.mark.gpu
def test_sharded_step_overflow_redo_equals_roomy_run():
    """rasterizer_view_grad_fn reuses one pair capacity across views without
    host syncs and redoes the step when a view overflowed it
    (check_overflow).  A step whose first view sees nothing (capacity sized
    from it, then forced small) and whose later views overflow must end with
    the same flat gradients, sigma signal and view counts as a step that had
    room from the start: the discarded attempt leaves no trace."""
    import paper_2411_14974_b200 as cs
    from paper_2411_14974_b200 import rasterizer as rz, synthetic
    arrays = synthetic.quantize32(synthetic.generate_scene(3000, seed=4))
    st = cs.SceneTensors.from_arrays(arrays, "cuda")
    tgt = cs.SceneTensors.from_arrays(synthetic.quantize32(synthetic.perturb(arrays, seed=6)), "cuda")
    W, H = 160, 120
    R, t = synthetic.look_at((0.0, 1.4, -4.0), target=(0.0, 1.4, -8.0))     # facing away: nothing visible
    away = cs.Camera(fx=100.0, fy=100.0, cx=W / 2, cy=H / 2, width=W, height=H, R=R, t=t)
    cams = [away] + synthetic.ring_cameras(3, W, H)
    views = [(c, cs.render(tgt, c).image) for c in cams]
    views = [(c, torch.tensor(im, dtype=torch.float32, device="cuda")) for c, im in views]
    mode, settings = cs.ScalingMode.DEPTH, cs.RenderSettings()

    def run(tight: bool):
        params = {k: getattr(st, k).clone() for k in sharded.PARAM_ORDER}
        scene = cs.SceneTensors(**{k: params[k] for k in ("points", "raw_delta", "raw_sigma", "raw_opacity",
                                                          "raw_mask", "sh")}, background=st.background)
        r = rz.Rasterizer("cuda")
        if tight:
            r._cap_hint[(scene.n, W, H)] = 1024          # the first (empty) view keeps the capacity tiny
        fn = sharded.rasterizer_view_grad_fn(scene, mode, settings, rasterizer=r)
        step = sharded.ViewShardedStep(params, sharded.StepConfig(), fn)
        calls = {"n": 0}
        inner = fn.check_overflow

        def counting(group=None):
            ovf = inner(group)
            calls["n"] += int(ovf)
            return ovf
        fn.check_overflow = counting
        step.step(views)
        return {k: v.clone() for k, v in step.flat.views.items()}, calls["n"]

    tight, redos = run(True)
    roomy, redos0 = run(False)
    assert redos >= 1 and redos0 == 0, (redos, redos0)
    torch.testing.assert_close(tight["sigma_views"], roomy["sigma_views"], rtol=0, atol=0)
    for k in list(sharded.PARAM_ORDER) + ["sigma_signal"]:
        a, b = tight[k].cpu().numpy().ravel(), roomy[k].cpu().numpy().ravel()
        scale = max(float(np.abs(b).max()), 1e-30)
        assert float(np.abs(a - b).max()) <= 1e-5 * scale, k     # float atomics: summation order only


def _mock_signal_fn(params, bucket_log=None):
    """A per-view function with the GPU function's interface (accumulates its
    own sigma signal; with ``ranges`` it hands every convex range on as soon
    as the range's rows are final, as the chain-per-range backward does)."""
    def fn(view, grads, signal, ranges=None, on_range=None):
        v = float(view)
        for name, g in grads.items():
            g.add_(torch.sin(params[name] * (1.0 + 0.1 * v) + v))
        n = params["points"].shape[0]
        vis = ((torch.arange(n) % (int(view) + 2)) != 0).to(grads["raw_sigma"].dtype)
        signal["sigma_signal"].add_(torch.cos(params["raw_sigma"] + v).abs() * vis)
        signal["sigma_views"].add_(vis)
        if ranges is not None:
            for first, last in ranges:
                if bucket_log is not None:
                    bucket_log.append((first, last))
                on_range(first, last)
        return torch.tensor(v)
    fn.handles_signal = True
    fn.supports_buckets = True
    return fn


def _bucket_worker(rank, world, port, out_path, buckets):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        params = _params()
        log = []
        step = sharded.ViewShardedStep(params, sharded.StepConfig(total_iterations=100),
                                       _mock_signal_fn(params, log), buckets=buckets)
        for _ in range(3):
            step.step(list(range(7)))
        torch.save({"params": params, "sigma": step.sigma_sum.clone(), "log": log}, f"{out_path}.{rank}")
    finally:
        dist.destroy_process_group()


def test_bucketed_all_reduce_equals_one_all_reduce():
    """the rank's last view hands its convex ranges to async
    all-reduces as their rows become final (overlapping the chain of the
    next range); the step ends bit-identical to one all-reduce of the whole
    buffer and to a single process."""
    results = {}
    for buckets in (1, 3):
        with tempfile.TemporaryDirectory() as tmp:
            out = os.path.join(tmp, "res")
            mp.spawn(_bucket_worker, args=(2, _free_port(), out, buckets), nprocs=2, join=True)
            results[buckets] = [torch.load(f"{out}.{r}") for r in range(2)]
    single = _params()
    step = sharded.ViewShardedStep(single, sharded.StepConfig(total_iterations=100), _mock_signal_fn(single))
    for _ in range(3):
        step.step(list(range(7)))
    r1, r3 = results[1], results[3]
    assert len(r3[0]["log"]) == 3 * 3 and r1[0]["log"] == [(0, 37)] * 3     # 3 ranges per step, 3 steps
    for name in single:
        torch.testing.assert_close(r3[0]["params"][name], r3[1]["params"][name], rtol=0, atol=0)
        torch.testing.assert_close(r3[0]["params"][name], r1[0]["params"][name], rtol=0, atol=0)
        torch.testing.assert_close(r3[0]["params"][name], single[name], rtol=1e-10, atol=1e-12)
    torch.testing.assert_close(r3[0]["sigma"], step.sigma_sum, rtol=1e-10, atol=1e-12)
