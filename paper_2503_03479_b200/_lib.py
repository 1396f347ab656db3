"""ctypes binding of libxa_b200.so (include/xaffine_b200.h).

The CUDA library is the only compute path: if it is missing this module
raises instead of falling back to anything on the CPU.
"""
from __future__ import annotations

import ctypes as C
import os
import pathlib
import threading

PKG = pathlib.Path(__file__).resolve().parent
# XA_LIB_PATH: load an A/B build variant (tools/build_variant.py) instead
LIB_PATH = pathlib.Path(os.environ.get("XA_LIB_PATH") or (PKG / "libxa_b200.so"))

XA_OK, XA_EINVAL, XA_ESINGULAR, XA_ECUDA, XA_ENOMEM, XA_ECAPACITY, XA_EPIPELINE, XA_EEVAL, XA_EIO = (
    0, -1, -2, -3, -4, -5, -6, -7, -8)
XA_EHOMOGRAPHY = -9
XA_U8, XA_F32 = 0, 1
XA_NEAREST, XA_LANCZOS = 0, 1


class XaKeypoint(C.Structure):
    _fields_ = [("x", C.c_float), ("y", C.c_float), ("response", C.c_float),
                ("orientation", C.c_float), ("octave_scale", C.c_float)]


class XaMatch(C.Structure):
    _fields_ = [("idx_a", C.c_int32), ("idx_b", C.c_int32), ("distance", C.c_float)]


class XaParams(C.Structure):
    _fields_ = [("psi", C.c_double), ("tilt", C.c_double), ("phi", C.c_double),
                ("scale", C.c_double), ("tx", C.c_double), ("ty", C.c_double)]


_lib = None
_lock = threading.Lock()

vp, i32, u64, f64, sz = C.c_void_p, C.c_int, C.c_uint64, C.c_double, C.c_size_t
_SIGS = {
    "xa_engine_create": (i32, [i32, C.POINTER(vp)]),
    "xa_engine_destroy": (i32, [vp]),
    "xa_last_error": (C.c_char_p, []),
    "xa_version": (i32, []),
    "xa_engine_stream": (vp, [vp]),
    "xa_engine_workspace_bytes": (sz, [vp]),
    "xa_engine_last_launches": (i32, [vp]),
    "xa_engine_read_pyramid": (i32, [vp, vp, C.c_size_t]),
    "xa_load_image": (i32, [C.c_char_p, vp, sz, vp, vp]),
    "xa_save_image": (i32, [vp, i32, i32, C.c_char_p]),
    "xa_save_png_rgb": (i32, [vp, i32, i32, C.c_char_p]),
    "xa_quantize": (i32, [vp, sz, vp]),
    "xa_fit_homography_dlt": (i32, [vp, i32, vp]),
    "xa_estimate_homography_ransac": (i32, [vp, i32, f64, i32, f64, u64, vp, vp, i32, vp]),
    "xa_engine_check": (i32, [vp]),
    "xa_engine_set_profiling": (i32, [vp, i32]),
    "xa_engine_orb_counters": (i32, [vp, i32, vp, C.POINTER(i32)]),
    "xa_engine_stage_times": (i32, [vp, i32, vp, vp, C.POINTER(i32)]),
    "xa_pattern_checksum": (u64, []),
    "xa_trig_fixups": (i32, []),
    "xa_simulation_from_params": (i32, [vp, vp]),
    "xa_affine_from_params": (i32, [vp, vp]),
    "xa_invert": (i32, [vp, vp]),
    "xa_build_param_grid": (i32, [f64, i32, f64, f64, vp, i32, C.POINTER(i32)]),
    "xa_warp_frame": (i32, [vp, i32, i32, C.POINTER(i32), C.POINTER(i32), C.POINTER(f64),
                            C.POINTER(f64), vp]),
    "xa_gaussian_blur": (i32, [vp, vp, i32, i32, f64, vp]),
    "xa_resize_bilinear": (i32, [vp, vp, i32, i32, i32, i32, vp]),
    "xa_antialias_tilt": (i32, [vp, vp, i32, i32, f64, f64, vp]),
    "xa_warp": (i32, [vp, i32, vp, i32, i32, vp, i32, vp, sz, C.POINTER(i32), C.POINTER(i32),
                      C.POINTER(f64), C.POINTER(f64), vp]),
    "xa_synth_warp_case": (i32, [vp, vp, i32, i32, vp, i32, vp, sz, C.POINTER(i32),
                                 C.POINTER(i32), vp]),
    "xa_detect_oriented_corners": (i32, [vp, vp, i32, i32, i32, vp, i32, C.POINTER(i32)]),
    "xa_describe_binary": (i32, [vp, vp, i32, i32, vp, i32, vp, vp, C.POINTER(i32)]),
    "xa_match_hamming": (i32, [vp, vp, i32, vp, i32, f64, vp, C.POINTER(i32)]),
    "xa_coarse_search": (i32, [vp, i32, vp, i32, i32, vp, i32, i32, vp, i32, i32, f64, i32, vp,
                               vp, vp]),
    "xa_coarse_search_device": (i32, [vp, i32, vp, i32, i32, vp, i32, i32, vp, i32, i32, f64,
                                      i32, vp, vp, vp]),
    "xa_coarse_search_batch": (i32, [vp, i32, vp, i32, i32, vp, i32, i32, i32, vp, i32, i32, f64,
                                     i32, vp, vp, vp]),
    "xa_coarse_search_batch_device": (i32, [vp, i32, vp, i32, i32, vp, i32, i32, i32, vp, i32, i32,
                                            f64, i32, vp, vp, vp]),
    "xa_coarse_search_multi": (i32, [vp, i32, i32, vp, i32, i32, vp, i32, i32, i32, vp, i32, i32,
                                     f64, i32, vp, vp, vp]),
    "xa_coarse_search_nccl": (i32, [vp, vp, i32, i32, i32, vp, i32, i32, vp, i32, i32, i32, vp, i32,
                                    i32, f64, i32, vp, vp, vp]),
    "xa_nccl_unique_id": (i32, [vp, sz]),
    "xa_nccl_comm_init": (i32, [C.POINTER(vp), i32, vp, i32, i32]),
    "xa_nccl_comm_destroy": (i32, [vp]),
    "xa_multi_last_error": (C.c_char_p, []),
    "xa_simulate_views_device": (i32, [vp, vp, i32, i32, vp, i32, i32, vp, vp, vp, vp,
                                       C.POINTER(sz), vp]),
    "xa_match_hamming_device": (i32, [vp, vp, i32, vp, i32, f64, vp, vp, vp, vp, vp]),
    "xa_match_ratio": (i32, [vp, vp, i32, vp, i32, f64, vp, C.POINTER(i32)]),
    "xa_detect_dog_keypoints": (i32, [vp, vp, i32, i32, i32, vp, i32, C.POINTER(i32)]),
    "xa_describe_gradient": (i32, [vp, vp, i32, i32, vp, i32, vp, vp, C.POINTER(i32)]),
    "xa_match_ratio_device": (i32, [vp, vp, i32, vp, i32, f64, vp, vp, vp, vp, vp]),
    "xa_asift_correspondences": (i32, [vp, vp, i32, i32, vp, i32, i32, vp, i32, i32, f64, i32,
                                       vp, i32, C.POINTER(i32)]),
}
EXPORTS = tuple(_SIGS)


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not LIB_PATH.exists():
                    raise ImportError(
                        f"{LIB_PATH} is missing: build it with "
                        "`python -m paper_2503_03479_b200.build` (there is no CPU fallback)")
                L = C.CDLL(str(LIB_PATH))
                for name, (res, args) in _SIGS.items():
                    fn = getattr(L, name)
                    fn.restype = res
                    fn.argtypes = args
                _lib = L
    return _lib


class XaError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def check(rc: int) -> None:
    if rc != XA_OK:
        raise XaError(rc, lib().xa_last_error().decode())
