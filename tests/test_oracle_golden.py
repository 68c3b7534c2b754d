"""Pin the CPU oracle (oracle/cs_oracle.c) to the reference's own outputs.

The fixtures come from running the reference package itself
(tests/golden/make_golden.py).  Discrete outputs (depth order, hull cycles,
bboxes, tile lists, counts, visibility) must be bit-exact; continuous ones
agree to float64 round-off (the reference uses NumPy's SIMD exp/log and BLAS,
the oracle glibc).
"""
import numpy as np
import pytest

import oracle
from tests import golden_cases as gc

CASES = gc.scene_cases()


def test_hull_cases_bit_exact():
    g = np.load(f"{gc.GOLDEN}/hulls.npz")
    pts, ns, hulls = g["points"], g["n"], g["hull"]
    for i in range(ns.size):
        got = oracle.graham_scan(pts[i, : ns[i]])
        want = hulls[i][hulls[i] >= 0]
        if want.size == 0:
            assert got is None, i
        else:
            assert got is not None, i
            np.testing.assert_array_equal(got, want, err_msg=f"hull case {i}")


@pytest.mark.parametrize("name", CASES)
def test_prepare_view_matches_reference(name):
    g = gc.load(name)
    view = oracle.prepare_view(gc.params(g), gc.camera(g), gc.settings(g))
    order = view["order"]
    np.testing.assert_array_equal(order, g["prep_index"])
    if order.size == 0:
        return
    k = g["points"].shape[1]
    hull = view["hull"][order]
    np.testing.assert_array_equal(np.where(hull >= 0, hull, -1), g["prep_hull"])
    np.testing.assert_array_equal(view["bbox"][order], g["prep_bbox"])
    # discrete-feeding quantities are reproduced exactly (pinned op order)
    np.testing.assert_array_equal(view["depth"][order], g["prep_depth"])
    np.testing.assert_array_equal(view["pixels"][order], g["prep_pixels"])
    mask = g["prep_hull"] >= 0
    np.testing.assert_array_equal(view["normals"][order][mask], g["prep_normals"][mask])
    np.testing.assert_array_equal(view["offsets"][order][mask], g["prep_offsets"][mask])
    np.testing.assert_allclose(view["delta_s"][order], g["prep_delta_s"], rtol=4e-16, atol=0)
    np.testing.assert_allclose(view["sigma_s"][order], g["prep_sigma_s"], rtol=4e-16, atol=0)
    np.testing.assert_allclose(view["opacity"][order], g["prep_opacity"], rtol=4e-16, atol=0)
    np.testing.assert_allclose(view["color"][order], g["prep_color"], rtol=0, atol=1e-14)
    assert k == view["hull"].shape[1]


@pytest.mark.parametrize("name", CASES)
def test_bin_tiles_match_reference(name):
    g = gc.load(name)
    cam, st = gc.camera(g), gc.settings(g)
    view = oracle.prepare_view(gc.params(g), cam, st)
    off, items = oracle.bin_tiles(view, cam["width"], cam["height"], st["tile"])
    np.testing.assert_array_equal(off, g["bin_offsets"])
    np.testing.assert_array_equal(items, g["bin_items"])


@pytest.mark.parametrize("name", CASES)
def test_render_matches_reference(name):
    g = gc.load(name)
    fr = oracle.render(gc.params(g), gc.camera(g), gc.settings(g))
    np.testing.assert_array_equal(fr["count"], g["count"])
    np.testing.assert_array_equal(fr["visible"], g["visible"])
    np.testing.assert_allclose(fr["image"], g["img"], rtol=0, atol=1e-12)
    np.testing.assert_allclose(fr["trans"], g["trans"], rtol=0, atol=1e-12)
    np.testing.assert_allclose(fr["wsum"], g["wsum"], rtol=0, atol=1e-12)
    if "ref_img" in g:   # render_reference == render(EXACT_SETTINGS)
        np.testing.assert_allclose(fr["image"], g["ref_img"], rtol=0, atol=1e-12)
        np.testing.assert_allclose(fr["trans"], g["ref_trans"], rtol=0, atol=1e-12)
        np.testing.assert_array_equal(fr["count"], g["ref_count"])


def grad_rel_error(a: np.ndarray, b: np.ndarray) -> float:
    """backward.py:464-467 relative error with its noise floor."""
    a, b = np.ravel(a), np.ravel(b)
    denom = np.maximum(np.abs(a), np.abs(b))
    if denom.size == 0 or denom.max() == 0:
        return 0.0
    floor = max(1e-6 * denom.max(), 1e-12)
    return float((np.abs(a - b) / np.maximum(denom, floor)).max())


@pytest.mark.parametrize("name", [c for c in CASES if "d_image" in gc.load(c)])
def test_backward_matches_reference(name):
    g = gc.load(name)
    gr = oracle.backward(gc.params(g), gc.camera(g), gc.settings(g), g["d_image"])
    np.testing.assert_array_equal(gr["visible"], g["g_visible"])
    for ours, theirs in (("d_points", "g_points"), ("d_raw_delta", "g_delta"),
                         ("d_raw_sigma", "g_sigma"), ("d_raw_opacity", "g_opacity"),
                         ("d_sh", "g_sh"), ("d_raw_mask", "g_mask")):
        err = grad_rel_error(gr[ours], g[theirs])
        assert err < 1e-8, (ours, err)


@pytest.mark.parametrize("name", [c for c in CASES if "d_image" in gc.load(c)])
def test_forced_backward_with_own_decisions_is_the_reference(name):
    """The decision-forced oracle backward (used to compare the GPU at its own
    discrete decisions) fed the reference's own decisions is the plain
    oracle backward, bit for bit; the decisions reproduce the counts."""
    g = gc.load(name)
    params, cam, st = gc.params(g), gc.camera(g), gc.settings(g)
    view = oracle.prepare_view(params, cam, st)
    tiles = oracle.bin_tiles(view, cam["width"], cam["height"], st["tile"])
    offsets, pos = oracle.blend_decisions(cam, st, view, tiles)
    np.testing.assert_array_equal(np.diff(offsets).reshape(g["count"].shape), g["count"])
    plain = oracle.backward(params, cam, st, g["d_image"], view=view, tiles=tiles)
    forced = oracle.backward(params, cam, st, g["d_image"], view=view, tiles=tiles, forced=(offsets, pos, None))
    for k in ("d_points", "d_raw_delta", "d_raw_sigma", "d_raw_opacity", "d_sh", "d_raw_mask"):
        np.testing.assert_array_equal(forced[k], plain[k], err_msg=k)


def test_forced_backward_follows_the_given_decisions():
    """Dropping one recorded blend from a pixel changes exactly the
    gradients of the convexes that pixel's walk reaches, and the forced walk
    takes it as given (a flipped threshold decision)."""
    g = gc.load("config1")
    params, cam, st = gc.params(g), gc.camera(g), gc.settings(g)
    view = oracle.prepare_view(params, cam, st)
    tiles = oracle.bin_tiles(view, cam["width"], cam["height"], st["tile"])
    offsets, pos = oracle.blend_decisions(cam, st, view, tiles)
    plain = oracle.backward(params, cam, st, g["d_image"], view=view, tiles=tiles)
    p = int(np.argmax(np.diff(offsets)))           # the pixel with the most blends
    drop = int(offsets[p]) + 2                      # its third blend
    off2 = offsets.copy()
    off2[p + 1:] -= 1
    pos2 = np.delete(pos, drop)
    forced = oracle.backward(params, cam, st, g["d_image"], view=view, tiles=tiles, forced=(off2, pos2, None))
    items = tiles[1]
    moved = np.flatnonzero(np.abs(forced["d_raw_opacity"] - plain["d_raw_opacity"]) > 0)
    # only convexes that pixel blended (at or before the dropped one, whose
    # transmittance / colour-behind terms change) can move
    blended = set(view["order"][items[pos[offsets[p]:offsets[p + 1]]]].tolist())
    assert moved.size > 0 and set(moved.tolist()) <= blended


@pytest.mark.parametrize("name", ["config1", "mode_none", "exact7", "alpha_cap"])
def test_forced_render_with_own_decisions_is_the_reference(name):
    """The decision-forced oracle render fed the reference's own decisions
    reproduces the plain render bit for bit."""
    g = gc.load(name)
    params, cam, st = gc.params(g), gc.camera(g), gc.settings(g)
    view = oracle.prepare_view(params, cam, st)
    tiles = oracle.bin_tiles(view, cam["width"], cam["height"], st["tile"])
    offsets, pos = oracle.blend_decisions(cam, st, view, tiles)
    plain = oracle.render(params, cam, st, view=view, tiles=tiles)
    forced = oracle.render(params, cam, st, view=view, tiles=tiles, forced=(offsets, pos))
    for k in ("image", "trans", "count", "wsum", "depth", "visible"):
        np.testing.assert_array_equal(forced[k], plain[k], err_msg=k)
