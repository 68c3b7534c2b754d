"""B200-native (sm_100a) 3D Convex Splatting rasterizer.

Drop-in for the hot path of the reference package ``convexsplat`` 0.1.0:
the names below mirror its public surface (``convexsplat/__init__.py``) for
the render / backward path.  The model types are importable without a GPU;
the renderer entry points need CUDA and the in-tree
``libconvexsplat_sm100.so`` (built by ``python -m paper_2411_14974_b200.build``).
"""
from .model import (ALPHA_MAX, EXACT_SETTINGS, MASK_GATE, MIN_POINTS, SH_COEFFS, TILE_SIZE, Camera,
                    GradientBuffer, RenderOutput, RenderSettings, ScalingMode, Scene, SmoothConvex,
                    delta_activation, inverse_delta_activation, inverse_mask_activation,
                    inverse_opacity_activation, inverse_sigma_activation, mask_activation,
                    opacity_activation, sigma_activation)

__version__ = "0.1.0"

_LAZY = {
    "SceneTensors": "scene_tensors", "as_scene_tensors": "scene_tensors",
    "render": "rasterizer", "render_reference": "rasterizer", "backward": "rasterizer",
    "prepare_view": "rasterizer", "bin_tiles": "rasterizer", "rasterize": "rasterizer",
    "Rasterizer": "rasterizer", "Workspace": "rasterizer", "inspect_frame": "rasterizer",
    "zero_grads": "rasterizer",
    "empty_grads": "rasterizer",
}


def __getattr__(name):  # torch-dependent modules load on first use
    mod = _LAZY.get(name)
    if mod is None:
        raise AttributeError(name)
    import importlib
    return getattr(importlib.import_module(f"{__name__}.{mod}"), name)


__all__ = sorted(["ALPHA_MAX", "EXACT_SETTINGS", "MASK_GATE", "MIN_POINTS", "SH_COEFFS", "TILE_SIZE", "Camera",
                  "GradientBuffer", "RenderOutput", "RenderSettings", "ScalingMode", "Scene", "SmoothConvex",
                  *_LAZY])
