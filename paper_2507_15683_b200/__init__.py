"""B200-native (sm_100a) 3DGS forward rasterizer -- the data-parallel hot path
of Hi^2-GSLoc (arXiv 2507.15683).  See include/gs.h and DESIGN.md.

The compute path is ``libgs.so`` (hand-written CUDA for sm_100a); this package
is the thin binding (``gs``), a buffer-managing batch harness (``pipeline``)
and the multi-GPU pose-sharding host logic (``dist``).  There is no CPU
fallback.
"""
from .gs import (GSError, DeviceScene, ViewBatch, Projected, Bins, Images, default_params,  # noqa: F401
                 gs_project, gs_bin_sort, gs_rasterize, gs_rasterize_backproject, gs_backproject, gs_visibility_score,
                 gs_validate_scene,
                 gs_match, Matches, match_workspace_bytes, gs_pnp, gs_verify_consistency, pnp_workspace_bytes,
                 ViewsAt, GS_VIEW_BYTES, gs_feature_backward, gs_feature_l1_grad, gs_feature_sgd, gs_radiance_backward, GRAD_FIELDS, gs_mean_backward,
                 gs_param_backward, gs_adam, gs_dssim_grad, gs_probe_alpha, gs_sanitize_scene, gs_joint_backward, gs_appearance_l1_grad, gs_pack_images,
                 gs_pack_bytes, unpack_dense11, GS_PACK_COMPACT, GS_PACK_DENSE11,
                 lib, LIB_PATH,
                 EXPORTS)
from .pipeline import Renderer, SignificanceScorer, Refiner, FeatureDistiller, SceneTrainer  # noqa: F401

__all__ = ["gs_project", "gs_bin_sort", "gs_rasterize", "gs_rasterize_backproject", "gs_backproject", "gs_visibility_score", "gs_match",
           "gs_validate_scene", "gs_pnp", "gs_verify_consistency", "Matches", "Refiner", "DeviceScene",
           "ViewBatch", "Projected", "Bins", "Images", "Renderer", "SignificanceScorer", "default_params", "GSError"]
