"""B200-native coarse pose search (affine view simulation -> ORB -> Hamming ratio
matching) of arXiv 2503.03479, behind the reference's xaffine interface.

The compute path is libxa_b200.so (hand-written sm_100a CUDA behind the C-ABI
in include/xaffine_b200.h); `api` mirrors the reference's function names.
"""
from . import api  # noqa: F401
from .api import (AffineParams, CoarseResult, Engine, GeometryError, GridConfig, ParamGrid,  # noqa: F401
                  PipelineError, WarpResult, affine_from_params, antialias_tilt,
                  build_param_grid, coarse_search, coarse_search_batch, coarse_search_multi,
                  coarse_search_nccl, describe_binary, describe_gradient, detect_dog_keypoints,
                  detect_oriented_corners,
                  gaussian_blur, hamming_distance, invert, map_point, match_hamming, match_ratio,
                  resize_bilinear, simulation_from_params, warp_lanczos, warp_nearest,
                  ReferenceDecision, filter_to_content, fine_correspondences, fine_features,
                  scaling_coefficient, select_reference, asift_correspondences,
                  EvalError, synth_warp_case, IoError, load_image, save_image, save_png_rgb, quantize,
                  HomographyError, fit_homography_dlt, estimate_homography_ransac)

__all__ = [n for n in dir(api) if not n.startswith("_")]
