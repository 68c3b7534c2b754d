"""ctypes binding of libconvexsplat_sm100.so (include/convexsplat_b200.h).

There is no CPU fallback: if the library is missing or cannot be loaded the
import of the renderer fails loudly.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libconvexsplat_sm100.so")

EXPORTS = ("cs_abi_version", "cs_error_string", "cs_workspace_layout", "cs_forward", "cs_backward",
           "cs_forward_stages", "cs_forward_ex", "cs_backward_stages", "cs_read_counters", "cs_graham_scan_batch",
           "cs_backward_signal", "cs_backward_ex", "cs_image_loss_workspace", "cs_image_loss", "cs_adam_step",
           "cs_checkpoint_unpack", "cs_checkpoint_pack", "cs_density_flags", "cs_density_scatter",
           "cs_read_status", "cs_forward_record", "cs_prepare_view_export", "cs_backward_chain_range",
           "cs_zero_accumulators")
ABI_VERSION = 8
ERR_WORKSPACE = 3     # CS_ERR_WORKSPACE
ERR_NONFINITE = 4     # CS_ERR_NONFINITE
ERR_UNSUPPORTED = 5   # CS_ERR_UNSUPPORTED
GRADS_OVERWRITE = 1   # CS_GRADS_OVERWRITE
WORK_COUNTERS = 2     # CS_WORK_COUNTERS
ACCUM_ZEROED = 4      # CS_ACCUM_ZEROED

_vp = ctypes.c_void_p


class CsCamera(ctypes.Structure):
    _fields_ = [("fx", ctypes.c_double), ("fy", ctypes.c_double), ("cx", ctypes.c_double),
                ("cy", ctypes.c_double), ("R", ctypes.c_double * 9), ("t", ctypes.c_double * 3),
                ("z_near", ctypes.c_double), ("width", ctypes.c_int32), ("height", ctypes.c_int32),
                ("ortho", ctypes.c_int32), ("reserved", ctypes.c_int32)]


class CsSettings(ctypes.Structure):
    _fields_ = [("cutoff", ctypes.c_double), ("floor", ctypes.c_double),
                ("background", ctypes.c_double * 3), ("tile", ctypes.c_int32),
                ("sh_degree", ctypes.c_int32), ("scaling_mode", ctypes.c_int32),
                ("reserved", ctypes.c_int32)]


class CsParams(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("k", ctypes.c_int32), ("reserved", ctypes.c_int32),
                ("points", _vp), ("raw_delta", _vp), ("raw_sigma", _vp), ("raw_opacity", _vp),
                ("raw_mask", _vp), ("sh", _vp)]


class CsFrame(ctypes.Structure):
    _fields_ = [("image", _vp), ("final_T", _vp), ("count", _vp), ("weight_sum", _vp),
                ("depth", _vp), ("visible", _vp)]


class CsGrads(ctypes.Structure):
    _fields_ = [("d_points", _vp), ("d_raw_delta", _vp), ("d_raw_sigma", _vp),
                ("d_raw_opacity", _vp), ("d_raw_mask", _vp), ("d_sh", _vp)]


class CsViewSignal(ctypes.Structure):
    _fields_ = [("sigma_signal", _vp), ("sigma_views", _vp), ("visible", _vp)]


class CsAdamTensor(ctypes.Structure):
    _fields_ = [("param", _vp), ("grad", _vp), ("m", _vp), ("v", _vp), ("numel", ctypes.c_int64),
                ("lr", ctypes.c_double)]


class CsSceneOut(ctypes.Structure):
    _fields_ = [("points", _vp), ("raw_delta", _vp), ("raw_sigma", _vp), ("raw_opacity", _vp),
                ("raw_mask", _vp), ("sh", _vp)]


class CsDensityConfig(ctypes.Structure):
    _fields_ = [("sigma_threshold", ctypes.c_double), ("split_scale", ctypes.c_double),
                ("split_sigma_boost", ctypes.c_double), ("split_opacity_factor", ctypes.c_double),
                ("prune_opacity", ctypes.c_double), ("size_limit", ctypes.c_double),
                ("allow_split", ctypes.c_int32), ("reserved", ctypes.c_int32)]


class CsViewExport(ctypes.Structure):
    _fields_ = [(name, _vp) for name in ("pixels", "point_depths", "normals", "offsets", "delta_s", "sigma_s",
                                         "opacity", "scale", "view_dir", "view_dist", "color")]


class CsLayout(ctypes.Structure):
    _fields_ = [(name, ctypes.c_size_t) for name in (
        "total_bytes", "counters", "records", "lines", "hull", "bbox", "depth_keys", "order", "tiles_touched",
        "pair_offsets", "pair_tiles", "pair_ids", "tile_ranges", "pixel_last", "pixel_T", "pixel_clamp",
        "grad_accum", "scratch", "scratch_bytes")] + [
        (name, ctypes.c_int32) for name in ("rec_floats", "acc_floats", "max_k", "tiles_x", "tiles_y",
                                            "reserved")]


class CsError(RuntimeError):
    pass


_lib = None


def load(path: str = None):
    """Load (once) and type the library.  Raises if it is absent.  CS_LIB_PATH
    overrides the in-tree library (used to A/B kernel variants)."""
    global _lib
    if _lib is not None:
        return _lib
    path = path or os.environ.get("CS_LIB_PATH") or LIB_PATH
    if not os.path.exists(path):
        raise CsError(f"{path} is missing: run `python -m paper_2411_14974_b200.build` "
                      "(there is no CPU fallback)")
    L = ctypes.CDLL(path)
    L.cs_abi_version.restype = ctypes.c_int
    L.cs_error_string.restype = ctypes.c_char_p
    L.cs_error_string.argtypes = [ctypes.c_int]
    L.cs_workspace_layout.argtypes = [ctypes.POINTER(CsCamera), ctypes.POINTER(CsSettings), ctypes.c_int64,
                                      ctypes.c_int32, ctypes.c_int64, ctypes.POINTER(CsLayout)]
    L.cs_forward.argtypes = [ctypes.POINTER(CsCamera), ctypes.POINTER(CsSettings), ctypes.POINTER(CsParams),
                             _vp, ctypes.c_size_t, ctypes.c_int64, ctypes.POINTER(CsFrame), _vp]
    L.cs_backward.argtypes = [ctypes.POINTER(CsCamera), ctypes.POINTER(CsSettings), ctypes.POINTER(CsParams),
                              _vp, ctypes.c_size_t, ctypes.c_int64, _vp, ctypes.POINTER(CsGrads), _vp]
    L.cs_forward_stages.argtypes = L.cs_forward.argtypes[:-1] + [ctypes.c_int32, ctypes.c_int32, _vp]
    L.cs_forward_ex.argtypes = L.cs_forward.argtypes[:-1] + [ctypes.c_uint32, ctypes.c_int32, ctypes.c_int32, _vp]
    L.cs_backward_stages.argtypes = L.cs_backward.argtypes[:-1] + [ctypes.c_int32, ctypes.c_int32, _vp]
    L.cs_read_counters.argtypes = [_vp, ctypes.POINTER(ctypes.c_uint32), _vp]
    L.cs_read_status.argtypes = [_vp, _vp]
    L.cs_forward_record.argtypes = L.cs_forward.argtypes[:-1] + [_vp, _vp, _vp]
    L.cs_backward_chain_range.argtypes = [ctypes.POINTER(CsCamera), ctypes.POINTER(CsSettings),
                                          ctypes.POINTER(CsParams), _vp, ctypes.c_size_t, ctypes.c_int64,
                                          ctypes.POINTER(CsGrads), ctypes.POINTER(CsViewSignal), ctypes.c_uint32,
                                          ctypes.c_int64, ctypes.c_int64, _vp]
    L.cs_zero_accumulators.argtypes = [ctypes.POINTER(CsCamera), ctypes.POINTER(CsSettings),
                                       ctypes.POINTER(CsParams), _vp, ctypes.c_size_t, ctypes.c_int64, _vp]
    L.cs_prepare_view_export.argtypes = [ctypes.POINTER(CsCamera), ctypes.POINTER(CsSettings),
                                         ctypes.POINTER(CsParams), _vp, ctypes.c_size_t, ctypes.c_int64,
                                         ctypes.POINTER(CsViewExport), _vp]
    L.cs_graham_scan_batch.argtypes = [ctypes.c_int32, ctypes.c_int32, _vp, _vp, _vp, _vp, _vp]
    L.cs_backward_signal.argtypes = L.cs_backward.argtypes[:-1] + [ctypes.POINTER(CsViewSignal), _vp]
    L.cs_backward_ex.argtypes = L.cs_backward.argtypes[:-1] + [ctypes.POINTER(CsViewSignal), ctypes.c_uint32,
                                                               ctypes.c_int32, ctypes.c_int32, _vp]
    L.cs_image_loss_workspace.argtypes = [ctypes.c_int32, ctypes.c_int32, ctypes.POINTER(ctypes.c_size_t)]
    L.cs_image_loss.argtypes = [ctypes.c_int32, ctypes.c_int32, _vp, _vp, _vp, ctypes.c_int64, ctypes.c_double,
                                ctypes.c_double, _vp, _vp, _vp, _vp, ctypes.c_size_t, _vp]
    L.cs_adam_step.argtypes = [ctypes.c_int32, ctypes.POINTER(CsAdamTensor), ctypes.c_double, ctypes.c_double,
                               ctypes.c_double, ctypes.c_int32, ctypes.c_double, _vp]
    L.cs_checkpoint_unpack.argtypes = [ctypes.c_int32, ctypes.c_int64, ctypes.c_int32, _vp,
                                       ctypes.POINTER(CsSceneOut), _vp]
    L.cs_checkpoint_pack.argtypes = [ctypes.c_int32, ctypes.c_int64, ctypes.c_int32, ctypes.POINTER(CsSceneOut),
                                     _vp, _vp]
    L.cs_density_flags.argtypes = [ctypes.POINTER(CsParams), _vp, ctypes.POINTER(CsDensityConfig), _vp, _vp, _vp,
                                   _vp, _vp]
    L.cs_density_scatter.argtypes = [ctypes.POINTER(CsParams), ctypes.POINTER(CsDensityConfig), _vp, _vp, _vp,
                                     _vp, _vp, ctypes.POINTER(CsSceneOut), _vp, _vp]
    for fn in ("cs_workspace_layout", "cs_forward", "cs_backward", "cs_forward_stages", "cs_forward_ex",
               "cs_backward_stages",
               "cs_read_counters", "cs_graham_scan_batch", "cs_backward_signal", "cs_backward_ex",
               "cs_image_loss_workspace",
               "cs_image_loss", "cs_adam_step", "cs_checkpoint_unpack", "cs_checkpoint_pack", "cs_density_flags",
               "cs_density_scatter", "cs_read_status", "cs_forward_record", "cs_prepare_view_export",
               "cs_backward_chain_range", "cs_zero_accumulators"):
        getattr(L, fn).restype = ctypes.c_int
    if L.cs_abi_version() != ABI_VERSION:
        raise CsError(f"ABI mismatch: library {L.cs_abi_version()} != {ABI_VERSION}")
    _lib = L
    return L


def check(rc: int, what: str):
    if rc != 0:
        raise CsError(f"{what}: {load().cs_error_string(rc).decode()} (code {rc})")
