"""CPU-side checks of the C ABI: the library loads, exports every entry point
declared in include/convexsplat_b200.h, and its host-only functions
(layout, argument validation, error strings) behave.  No kernel runs here."""
import ctypes
import os
import re

import numpy as np
import pytest

from paper_2411_14974_b200 import _lib, build
from paper_2411_14974_b200.model import Camera, RenderSettings, ScalingMode

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "convexsplat_b200.h")


@pytest.fixture(scope="module")
def lib():
    build.build()
    return _lib.load()


def declared_functions():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"CS_API\s+[\w\s\*]*?\b(cs_\w+)\s*\(", text)))


def test_header_declares_the_bound_entry_points():
    assert declared_functions() == sorted(_lib.EXPORTS)


def test_library_exports_every_declared_symbol(lib):
    for name in declared_functions():
        assert hasattr(lib, name), name
    assert lib.cs_abi_version() == _lib.ABI_VERSION


def test_struct_sizes_match_the_header(lib):
    # the C structs are plain doubles / int32 / pointers with natural alignment
    assert ctypes.sizeof(_lib.CsCamera) == 8 * (4 + 9 + 3 + 1) + 4 * 4
    assert ctypes.sizeof(_lib.CsSettings) == 8 * 5 + 4 * 4
    assert ctypes.sizeof(_lib.CsParams) == 8 + 4 + 4 + 6 * 8
    assert ctypes.sizeof(_lib.CsFrame) == 6 * 8
    assert ctypes.sizeof(_lib.CsGrads) == 6 * 8


def _structs(width=1920, height=1080, settings=RenderSettings()):
    from paper_2411_14974_b200.rasterizer import camera_struct, settings_struct
    cam = Camera(fx=1000.0, fy=1000.0, cx=width / 2, cy=height / 2, width=width, height=height,
                 R=np.eye(3), t=np.array([0.0, 0.0, 4.0]))
    return camera_struct(cam), settings_struct(settings, ScalingMode.DEPTH, np.zeros(3))


def test_workspace_layout_regions_are_disjoint_and_aligned(lib):
    cam, st = _structs()
    L = _lib.CsLayout()
    assert lib.cs_workspace_layout(ctypes.byref(cam), ctypes.byref(st), 1_000_000, 6, 8_000_000,
                                   ctypes.byref(L)) == 0
    assert (L.tiles_x, L.tiles_y) == (120, 68)
    assert L.max_k == 8 and L.rec_floats == 16 and L.acc_floats == 32
    names = ["counters", "records", "lines", "hull", "bbox", "depth_keys", "order", "tiles_touched", "pair_offsets",
             "pair_tiles", "pair_ids", "tile_ranges", "pixel_last", "pixel_T", "pixel_clamp", "grad_accum",
             "scratch"]
    offs = [getattr(L, n) for n in names]
    assert offs == sorted(offs)
    assert all(o % 256 == 0 for o in offs)
    assert L.total_bytes >= L.scratch + L.scratch_bytes
    assert L.pair_ids - L.pair_tiles >= 4 * 8_000_000


def test_layout_rejects_bad_arguments(lib):
    cam, st = _structs()
    L = _lib.CsLayout()
    assert lib.cs_workspace_layout(ctypes.byref(cam), ctypes.byref(st), 10, 2, 100, ctypes.byref(L)) == 1  # K < 3
    assert lib.cs_workspace_layout(ctypes.byref(cam), ctypes.byref(st), 10, 17, 100, ctypes.byref(L)) == 1
    assert lib.cs_workspace_layout(ctypes.byref(cam), ctypes.byref(st), -1, 6, 100, ctypes.byref(L)) == 1
    cam8, st8 = _structs(settings=RenderSettings(tile_size=8))
    assert lib.cs_workspace_layout(ctypes.byref(cam8), ctypes.byref(st8), 10, 6, 100, ctypes.byref(L)) == _lib.ERR_UNSUPPORTED
    camd, std = _structs(settings=RenderSettings(sh_degree=4))
    assert lib.cs_workspace_layout(ctypes.byref(camd), ctypes.byref(std), 10, 6, 100, ctypes.byref(L)) == _lib.ERR_UNSUPPORTED


def test_forward_rejects_small_workspace_without_touching_the_gpu(lib):
    cam, st = _structs(64, 64)
    p = _lib.CsParams()
    p.n, p.k = 0, 6
    f = _lib.CsFrame(1, 1, 1, 1, 0, 0)   # non-null dummies: validation happens before any launch
    rc = lib.cs_forward(ctypes.byref(cam), ctypes.byref(st), ctypes.byref(p), ctypes.c_void_p(1), 16, 0,
                        ctypes.byref(f), None)
    assert rc == 3


def test_error_strings(lib):
    for code in range(6):
        assert lib.cs_error_string(code)
    assert b"unknown" in lib.cs_error_string(99)


def test_training_and_scene_structs_match_the_header(lib):
    assert ctypes.sizeof(_lib.CsViewSignal) == 3 * 8
    assert ctypes.sizeof(_lib.CsAdamTensor) == 4 * 8 + 8 + 8
    assert ctypes.sizeof(_lib.CsSceneOut) == 6 * 8
    assert ctypes.sizeof(_lib.CsDensityConfig) == 6 * 8 + 2 * 4


def test_training_entry_points_validate_before_launching(lib):
    """Argument checks of cs_image_loss / cs_adam_step / cs_checkpoint_* /
    cs_density_* run on the host (no device needed): losses.py:60-63 size
    check, precision 16|32, K range, null pointers."""
    size = ctypes.c_size_t()
    assert lib.cs_image_loss_workspace(10, 40, ctypes.byref(size)) == 1
    assert lib.cs_image_loss_workspace(70, 100, ctypes.byref(size)) == 0
    assert size.value == 4 * 9 * 60 * 90
    one = ctypes.c_void_p(1)
    assert lib.cs_image_loss(70, 100, None, one, one, 3, 0.2, 5e-4, one, one, one, one, size.value, None) == 1
    assert lib.cs_image_loss(70, 100, one, one, one, 3, 0.2, 5e-4, one, one, one, one, size.value - 4, None) == 3
    assert lib.cs_adam_step(9, None, 0.9, 0.999, 1e-15, 1, 1.0, None) == 1
    t = (_lib.CsAdamTensor * 1)()
    assert lib.cs_adam_step(1, t, 0.9, 0.999, 1e-15, 0, 1.0, None) == 1        # step counts from 1
    assert lib.cs_adam_step(0, t, 0.9, 0.999, 1e-15, 1, 1.0, None) == 0        # nothing to do
    out = _lib.CsSceneOut()
    assert lib.cs_checkpoint_unpack(8, 1, 6, one, ctypes.byref(out), None) == 1
    assert lib.cs_checkpoint_unpack(32, 1, 2, one, ctypes.byref(out), None) == 1
    assert lib.cs_checkpoint_pack(16, 1, 6, ctypes.byref(out), one, None) == 1   # null arrays
    assert lib.cs_checkpoint_unpack(16, 0, 6, None, None, None) == 0              # empty scene
    p = _lib.CsParams()
    p.n, p.k = 0, 6
    cfg = _lib.CsDensityConfig()
    assert lib.cs_density_flags(ctypes.byref(p), None, None, None, None, None, None, None) == 1
    assert lib.cs_density_flags(ctypes.byref(p), None, ctypes.byref(cfg), None, None, None, None, None) == 0
    assert lib.cs_abi_version() == _lib.ABI_VERSION == 8
    # cs_zero_accumulators validates before launching
    assert lib.cs_zero_accumulators(None, None, None, None, 0, 0, None) == 1


def test_backward_ex_validates_flags_and_signal(lib):
    """cs_backward_ex: unknown flag bits and a signal with null arrays are
    argument errors (checked before any launch)."""
    cam, st = _lib.CsCamera(), _lib.CsSettings()
    cam.width, cam.height, cam.fx, cam.fy = 64, 48, 50.0, 50.0
    st.tile, st.sh_degree = 16, 3
    p = _lib.CsParams()
    p.n, p.k = 0, 6
    g = _lib.CsGrads()
    one = ctypes.c_void_p(1)
    args = (ctypes.byref(cam), ctypes.byref(st), ctypes.byref(p), one, 1 << 30, 0, one, ctypes.byref(g))
    assert lib.cs_backward_ex(*args, None, 8, 0, 1, None) == 1                     # unknown flag
    sig = _lib.CsViewSignal(None, None, None)
    assert lib.cs_backward_ex(*args, ctypes.byref(sig), 0, 0, 1, None) == 1        # null signal arrays
    assert lib.cs_backward_ex(*args, None, 1, 1, 0, None) == 1                     # stages out of order
    fr = _lib.CsFrame()
    fargs = (ctypes.byref(cam), ctypes.byref(st), ctypes.byref(p), one, 1 << 30, 0, ctypes.byref(fr))
    assert lib.cs_forward_ex(*fargs, 4, 0, 2, None) == 1                            # unknown flag
    assert lib.cs_forward_ex(*fargs, 2, 2, 1, None) == 1                            # stages out of order
