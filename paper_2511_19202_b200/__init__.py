"""B200-native instanced 3DGS renderer with neural occlusion culling.

Drop-in for the reference ``splatcull`` render path (arXiv 2511.19202
desk-scale package): same public names (reference sc/__init__.py:3-29) plus
the SPEC-level scene / visibility-MLP API, computed by hand-written sm_100a
kernels in ``libsplatcull_b200.so`` (see include/splatcull_b200.h).
Importing the package needs no GPU; rendering does, and raises without one.
"""

from .asset import (Asset, Gaussian, asset_hash, compute_sampling_distances, logit, prepare, prune, recenter,
                    sigmoid, validate_asset)
from .camera import Camera, diag_to_fov_y, fov_y_to_diag, train_focal
from .nn import Mlp, VisibilityModel, encode_features, forward, init_mlp, load_model, make_model, save_model
from .layout import load_scene, orbit_eval, save_scene
from .ply import load_ply, save_ply
from .raster import RenderOutput, compute_metrics_pair, psnr, render, ssim
from .scene import (ComposedScene, FrameStats, InstanceTransform, Renderer, RenderOptions, local_inputs,
                    render_composed, render_path)
from .training import TrainConfig, evaluate, grad_check, lr_at, train

__all__ = [
    "Asset", "Gaussian", "Camera", "RenderOutput", "asset_hash", "compute_metrics_pair", "load_ply", "save_ply",
    "compute_sampling_distances", "prepare", "prune", "recenter", "render", "sigmoid", "logit",
    "validate_asset", "diag_to_fov_y", "fov_y_to_diag", "train_focal", "psnr", "ssim",
    "Mlp", "VisibilityModel", "init_mlp", "make_model", "forward", "encode_features",
    "ComposedScene", "InstanceTransform", "FrameStats", "RenderOptions", "Renderer", "render_composed",
    "local_inputs", "render_path", "save_model", "load_model", "TrainConfig", "train", "load_scene", "save_scene", "orbit_eval", "evaluate", "grad_check", "lr_at",
]

__version__ = "0.1.0"
