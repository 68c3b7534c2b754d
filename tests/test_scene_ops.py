"""Checkpoint I/O (sceneio.py:251-320) and densify/prune (density.py:54-105)
on the SoA tensors, against files and results produced by the reference
(tests/golden/make_golden.py gen_scene_ops)."""
import os
import shutil
import struct

import numpy as np
import pytest
import torch

from tests import golden_cases as gc

FIELDS = ("points", "raw_delta", "raw_sigma", "raw_opacity", "raw_mask", "sh")


def _io():
    from paper_2411_14974_b200 import scene_io
    return scene_io


def _corrupt(tmp_path, name, edit):
    raw = bytearray(open(os.path.join(gc.GOLDEN, "ckpt_f32.3dcs"), "rb").read())
    edit(raw)
    p = tmp_path / name
    p.write_bytes(bytes(raw))
    return p


def test_header_validation_matches_reference_errors(tmp_path):
    """The checks and their order of sceneio.load_checkpoint (sceneio.py:282-301)."""
    io = _io()
    ok = open(os.path.join(gc.GOLDEN, "ckpt_f32.3dcs"), "rb").read()
    h = io.read_header(ok)
    assert (h["precision"], h["count"], h["k"]) == (32, 9, 6)
    g = np.load(os.path.join(gc.GOLDEN, "ckpt.npz"))
    np.testing.assert_array_equal(h["background"], g["background"])
    assert h["scene_extent"] == float(g["scene_extent"])
    cases = {
        "short": (lambda r: r.__delitem__(slice(10, None)), "too small"),
        "magic": (lambda r: r.__setitem__(slice(0, 4), b"XXXX"), "bad magic"),
        "version": (lambda r: r.__setitem__(slice(4, 8), struct.pack("<I", 2)), "unsupported version"),
        "precision": (lambda r: r.__setitem__(slice(8, 12), struct.pack("<I", 8)), "bad precision"),
        "size": (lambda r: r.extend(b"\0\0\0\0"), "payload is"),
    }
    for name, (edit, msg) in cases.items():
        p = _corrupt(tmp_path, name, edit)
        with pytest.raises(io.CheckpointFormatError, match=msg):
            io.read_header(p.read_bytes(), p)
    assert issubclass(io.CheckpointFormatError, ValueError)


@pytest.mark.gpu
@pytest.mark.parametrize("prec", [32, 16])
def test_checkpoint_load_and_save_match_reference(tmp_path, prec):
    io = _io()
    g = np.load(os.path.join(gc.GOLDEN, "ckpt.npz"))
    src = os.path.join(gc.GOLDEN, f"ckpt_f{prec}.3dcs")
    st = io.load_checkpoint(src, "cuda")
    for f in FIELDS:
        want = g[f].astype(np.float32)
        if prec == 16:
            want = want.astype(np.float16).astype(np.float32)   # sceneio: rows.astype('<f2')
        np.testing.assert_array_equal(getattr(st, f).cpu().numpy(), want, err_msg=f)
    np.testing.assert_array_equal(st.background, g["background"])
    assert st.scene_extent == float(g["scene_extent"])
    # save the float32 scene back: byte-identical to the reference writer
    full = io.load_checkpoint(os.path.join(gc.GOLDEN, "ckpt_f32.3dcs"), "cuda")
    out = tmp_path / "out.3dcs"
    io.save_checkpoint(out, full, precision=prec)
    assert out.read_bytes() == open(src, "rb").read()


def test_checkpoint_save_rejects_bad_precision_and_empty(tmp_path):
    io = _io()
    from paper_2411_14974_b200.scene_tensors import SceneTensors
    empty = SceneTensors(torch.zeros(0, 6, 3), torch.zeros(0), torch.zeros(0), torch.zeros(0), torch.zeros(0),
                         torch.zeros(0, 16, 3))
    with pytest.raises(ValueError):
        io.save_checkpoint(tmp_path / "x.3dcs", empty, precision=8)
    with pytest.raises(ValueError):
        io.save_checkpoint(tmp_path / "x.3dcs", empty, precision=32)


@pytest.mark.gpu
@pytest.mark.parametrize("tag", ["split", "nosplit"])
def test_densify_and_prune_matches_reference(tag):
    """Split + prune (iteration 600) and prune only (after densify_stop):
    same rows in the same order, same index map and statistics."""
    from paper_2411_14974_b200 import density
    from paper_2411_14974_b200.scene_tensors import SceneTensors
    g = np.load(os.path.join(gc.GOLDEN, "density.npz"))
    st = SceneTensors.from_arrays({f: g[f"in_{f}"] for f in FIELDS}, "cuda", scene_extent=float(g["scene_extent"]))
    signal = torch.tensor(g["signal"], dtype=torch.float32)
    new, index_map, stats = density.densify_and_prune(st, signal, density.DensityConfig(), int(g[f"{tag}_iteration"]))
    np.testing.assert_array_equal(index_map.cpu().numpy(), g[f"{tag}_index_map"])
    assert [stats.split, stats.pruned, stats.before, stats.after] == list(g[f"{tag}_stats"])
    for f in FIELDS:
        got = getattr(new, f).cpu().numpy()
        want = g[f"{tag}_{f}"].astype(np.float32)     # reference float64 children, rounded to float32
        np.testing.assert_array_equal(got, want, err_msg=f)
    assert new.scene_extent == st.scene_extent


@pytest.mark.gpu
def test_sharded_step_densify_rebuilds_state():
    """ViewShardedStep.densify: new rows, remapped Adam moments (survivors keep
    theirs, children start at zero), fresh buffers sized for the new scene."""
    import paper_2411_14974_b200 as cs
    from paper_2411_14974_b200 import sharded, synthetic
    arrays = synthetic.quantize32(synthetic.generate_scene(500, seed=9))
    st = cs.SceneTensors.from_arrays(arrays, "cuda", scene_extent=2.0)
    cams = synthetic.ring_cameras(2, 64, 48)
    tgt = cs.SceneTensors.from_arrays(synthetic.quantize32(synthetic.perturb(arrays, seed=2)), "cuda")
    views = [(c, torch.tensor(cs.render(tgt, c).image, dtype=torch.float32, device="cuda")) for c in cams]
    mode, settings = cs.ScalingMode.DEPTH, cs.RenderSettings()
    params = {k: getattr(st, k) for k in sharded.PARAM_ORDER}
    step = sharded.ViewShardedStep(params, sharded.StepConfig(), sharded.rasterizer_view_grad_fn(st, mode, settings))
    step.step(views)
    m_before = step.adam.m["raw_delta"].clone()
    from paper_2411_14974_b200.density import DensityConfig
    new = step.densify(st, DensityConfig(sigma_loss_threshold=0.0))   # everything visible splits
    stats = step.last_densify
    assert stats.before == 500 and stats.after == new.n and stats.split > 0
    assert step.flat.views["points"].shape == new.points.shape
    assert step.adam.m["raw_delta"].shape[0] == new.n
    # continue training on the new scene
    step.view_grad_fn = sharded.rasterizer_view_grad_fn(new, mode, settings)
    step.step(views)
    assert torch.isfinite(step.flat.buffer).all()
    del m_before
