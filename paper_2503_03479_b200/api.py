"""Python mirror of the reference's hot-path interface, backed by the B200 library.

Names, argument meaning and error behaviour follow namespace xaffine in
proj/include/xaffine/*.hpp of the reference:

  geometry.hpp  AffineParams, GridConfig, ParamGrid, affine_from_params,
                simulation_from_params, invert, map_point, build_param_grid
  image.hpp     gaussian_blur, resize_bilinear (GrayImage = 2-D float32 array)
  warp.hpp      WarpResult, warp_nearest, warp_lanczos, antialias_tilt
  features.hpp  Keypoint (KEYPOINT dtype), BinaryDescriptor ((n, 4) uint64),
                MatchPair (MATCH dtype), hamming_distance
  orb.hpp       detect_oriented_corners, describe_binary, match_hamming
  pipeline.hpp  CoarseResult, coarse_search, PipelineError

Every computation runs in libxa_b200.so (sm_100a kernels behind the C-ABI in
include/xaffine_b200.h); only the reference's host-side geometry (a few double
multiplies per view) runs on the CPU, inside that same library.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import math
import threading
from typing import List, Sequence, Tuple

import numpy as np

from . import _lib
from ._lib import XA_F32, XA_LANCZOS, XA_NEAREST, XA_U8, XaError, XaKeypoint, XaMatch, XaParams

KEYPOINT = np.dtype([("x", "<f4"), ("y", "<f4"), ("response", "<f4"), ("orientation", "<f4"),
                     ("octave_scale", "<f4")])
MATCH = np.dtype([("idx_a", "<i4"), ("idx_b", "<i4"), ("distance", "<f4")])


class GeometryError(ValueError):
    """xaffine::GeometryError (geometry.hpp:11-13)."""


class PipelineError(RuntimeError):
    """xaffine::PipelineError (pipeline.hpp:16-18)."""


class EvalError(RuntimeError):
    """xaffine::EvalError (eval.hpp:14-16)."""


class IoError(RuntimeError):
    """xaffine::IoError (image_io.hpp:10-12)."""


class HomographyError(RuntimeError):
    """xaffine::HomographyError (homography.hpp:11-13)."""


def _check(rc: int) -> None:
    if rc == _lib.XA_OK:
        return
    msg = _lib.lib().xa_last_error().decode()
    if rc in (_lib.XA_EINVAL, _lib.XA_ESINGULAR) and ("tilt" in msg or "scale" in msg
                                                       or "singular" in msg or "grid" in msg
                                                       or "build_param_grid" in msg):
        raise GeometryError(msg)
    if rc == _lib.XA_EPIPELINE:
        raise PipelineError(msg)
    if rc == _lib.XA_EEVAL:
        raise EvalError(msg)
    if rc == _lib.XA_EIO:
        raise IoError(msg)
    if rc == _lib.XA_EHOMOGRAPHY:
        raise HomographyError(msg)
    if rc == _lib.XA_ESINGULAR:
        raise GeometryError(msg)
    raise XaError(rc, msg)


# ------------------------------------------------------------------ engine

class Engine:
    """One device context: CUDA stream + grow-only workspace (not thread-safe)."""

    def __init__(self, device: int = 0):
        L = _lib.lib()
        h = C.c_void_p()
        _check(L.xa_engine_create(device, C.byref(h)))
        self.handle = h
        self.device = device

    def close(self):
        if self.handle:
            _lib.lib().xa_engine_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def stream(self) -> int:
        return int(_lib.lib().xa_engine_stream(self.handle) or 0)

    def last_launches(self) -> int:
        return int(_lib.lib().xa_engine_last_launches(self.handle))

    def workspace_bytes(self) -> int:
        return int(_lib.lib().xa_engine_workspace_bytes(self.handle))

    def check(self) -> None:
        _check(_lib.lib().xa_engine_check(self.handle))

    def set_profiling(self, on: bool) -> None:
        _check(_lib.lib().xa_engine_set_profiling(self.handle, 1 if on else 0))

    def orb_counters(self, n_images: int) -> np.ndarray:
        """(n, 5) int32: candidates, thr-20 survivors, thr-7 survivors (auto-relaxed images
        only), detected, described."""
        out = np.zeros((max(n_images, 1), 5), np.int32)
        n = C.c_int()
        _check(_lib.lib().xa_engine_orb_counters(self.handle, n_images, out.ctypes.data_as(C.c_void_p),
                                                 C.byref(n)))
        return out[:n.value]

    def stage_times(self) -> List[Tuple[str, float]]:
        """Per-stage device milliseconds of the last profiled call (CUDA events)."""
        cap = 4096  # a batched call records 9 marks per chunk
        ms = (C.c_float * cap)()
        names = (C.c_char_p * cap)()
        n = C.c_int()
        _check(_lib.lib().xa_engine_stage_times(self.handle, cap, ms, names, C.byref(n)))
        return [(names[i].decode(), float(ms[i])) for i in range(n.value)]

    # ---- device-resident entry points (pointers are device addresses) ----
    def coarse_search_device(self, pixel_type, d_ref, w, h, d_target, tw, th, grid,
                             max_points, ratio, warp_mode, d_counts, d_kp_counts=0, stream=0):
        params = _params_array(grid)
        _check(_lib.lib().xa_coarse_search_device(
            self.handle, pixel_type, C.c_void_p(d_ref), w, h, C.c_void_p(d_target), tw, th,
            params, len(params), max_points, ratio, warp_mode, C.c_void_p(d_counts),
            C.c_void_p(d_kp_counts or None), C.c_void_p(stream or None)))

    def coarse_search_batch_device(self, pixel_type, d_refs, w, h, d_targets, tw, th, grid,
                                   max_points, ratio, warp_mode, d_counts, d_kp_counts=0,
                                   stream=0):
        """d_refs / d_targets: sequences of device addresses (one per pair);
        d_counts / d_kp_counts: device int32[len(d_refs) * len(grid)]."""
        params = _params_array(grid)
        P = len(d_refs)
        R = (C.c_void_p * P)(*[C.c_void_p(int(x)) for x in d_refs])
        T = (C.c_void_p * P)(*[C.c_void_p(int(x)) for x in d_targets])
        _check(_lib.lib().xa_coarse_search_batch_device(
            self.handle, pixel_type, R, w, h, T, tw, th, P, params, len(params), max_points, ratio,
            warp_mode, C.c_void_p(d_counts), C.c_void_p(d_kp_counts or None),
            C.c_void_p(stream or None)))

    def simulate_views_plan(self, w, h, views, warp_mode):
        params = _params_array(views)
        n = len(params)
        offs = np.zeros(n, np.int64)
        ws = np.zeros(n, np.int32)
        hs = np.zeros(n, np.int32)
        total = C.c_size_t()
        _check(_lib.lib().xa_simulate_views_device(
            self.handle, None, w, h, params, n, warp_mode, None, offs.ctypes.data_as(C.c_void_p),
            ws.ctypes.data_as(C.c_void_p), hs.ctypes.data_as(C.c_void_p), C.byref(total), None))
        return offs, ws, hs, total.value

    def simulate_views_device(self, d_src, w, h, views, warp_mode, d_out, stream=0):
        params = _params_array(views)
        n = len(params)
        offs = np.zeros(n, np.int64)
        ws = np.zeros(n, np.int32)
        hs = np.zeros(n, np.int32)
        total = C.c_size_t()
        _check(_lib.lib().xa_simulate_views_device(
            self.handle, C.c_void_p(d_src), w, h, params, n, warp_mode, C.c_void_p(d_out),
            offs.ctypes.data_as(C.c_void_p), ws.ctypes.data_as(C.c_void_p),
            hs.ctypes.data_as(C.c_void_p), C.byref(total), C.c_void_p(stream or None)))
        return offs, ws, hs

    def match_ratio_device(self, d_a, na, d_b, nb, ratio, d_best_idx, d_dist, d_keep, d_count,
                           stream=0):
        _check(_lib.lib().xa_match_ratio_device(
            self.handle, C.c_void_p(d_a), na, C.c_void_p(d_b), nb, ratio, C.c_void_p(d_best_idx),
            C.c_void_p(d_dist), C.c_void_p(d_keep), C.c_void_p(d_count), C.c_void_p(stream or None)))

    def match_hamming_device(self, d_a, na, d_b, nb, ratio, d_best_idx, d_best, d_second,
                             d_count, stream=0):
        _check(_lib.lib().xa_match_hamming_device(
            self.handle, C.c_void_p(d_a), na, C.c_void_p(d_b), nb, ratio,
            C.c_void_p(d_best_idx), C.c_void_p(d_best), C.c_void_p(d_second),
            C.c_void_p(d_count), C.c_void_p(stream or None)))


_tls = threading.local()


def default_engine(device: int = 0) -> Engine:
    """Per-thread engine (the reference calls the hot path from parallel_for workers)."""
    engines = getattr(_tls, "engines", None)
    if engines is None:
        engines = _tls.engines = {}
    if device not in engines:
        engines[device] = Engine(device)
    return engines[device]


# ------------------------------------------------------------------ geometry

@dataclasses.dataclass
class AffineParams:
    """xaffine::AffineParams (geometry.hpp:34-41)."""
    psi: float = 0.0
    tilt: float = 1.0
    phi: float = 0.0
    scale: float = 1.0
    tx: float = 0.0
    ty: float = 0.0

    def as_tuple(self):
        return (self.psi, self.tilt, self.phi, self.scale, self.tx, self.ty)


@dataclasses.dataclass
class GridConfig:
    """xaffine::GridConfig (geometry.hpp:44-49)."""
    a: float = math.sqrt(2.0)
    n: int = 5
    b_deg: float = 72.0
    delta_s: float = 0.5


@dataclasses.dataclass
class ParamGrid:
    entries: List[AffineParams]
    config: GridConfig


def _params_array(entries) -> "C.Array":
    if isinstance(entries, ParamGrid):
        entries = entries.entries
    arr = (XaParams * len(entries))()
    for i, p in enumerate(entries):
        t = p.as_tuple() if isinstance(p, AffineParams) else tuple(float(v) for v in p)
        arr[i] = XaParams(*t)
    return arr


def _mat(m) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(m, np.float64).reshape(9))


def affine_from_params(p: AffineParams) -> np.ndarray:
    out = np.zeros(9, np.float64)
    _check(_lib.lib().xa_affine_from_params(C.byref(XaParams(*p.as_tuple())),
                                            out.ctypes.data_as(C.c_void_p)))
    return out.reshape(3, 3)


def simulation_from_params(p: AffineParams) -> np.ndarray:
    out = np.zeros(9, np.float64)
    _check(_lib.lib().xa_simulation_from_params(C.byref(XaParams(*p.as_tuple())),
                                                out.ctypes.data_as(C.c_void_p)))
    return out.reshape(3, 3)


def invert(m) -> np.ndarray:
    a = _mat(m)
    out = np.zeros(9, np.float64)
    _check(_lib.lib().xa_invert(a.ctypes.data_as(C.c_void_p), out.ctypes.data_as(C.c_void_p)))
    return out.reshape(3, 3)


def map_point(m, x: float, y: float) -> Tuple[float, float]:
    """geometry.cpp:80-82 (same evaluation order)."""
    m = _mat(m)
    return (m[0] * x + m[1] * y + m[2], m[3] * x + m[4] * y + m[5])


def build_param_grid(cfg: GridConfig = GridConfig()) -> ParamGrid:
    n = C.c_int()
    _check(_lib.lib().xa_build_param_grid(cfg.a, cfg.n, cfg.b_deg, cfg.delta_s, None, 0,
                                          C.byref(n)))
    arr = (XaParams * max(n.value, 1))()
    _check(_lib.lib().xa_build_param_grid(cfg.a, cfg.n, cfg.b_deg, cfg.delta_s, arr, n.value,
                                          C.byref(n)))
    entries = [AffineParams(a.psi, a.tilt, a.phi, a.scale, a.tx, a.ty) for a in arr[:n.value]]
    return ParamGrid(entries, cfg)


# ------------------------------------------------------------------ images

def _img(img) -> np.ndarray:
    a = np.ascontiguousarray(img, dtype=np.float32)
    if a.ndim != 2:
        raise ValueError("GrayImage must be a 2-D array (height, width)")
    return a


def _ptr(a: np.ndarray) -> C.c_void_p:
    return a.ctypes.data_as(C.c_void_p)


def gaussian_blur(img, sigma: float, engine: Engine = None) -> np.ndarray:
    a = _img(img)
    e = engine or default_engine()
    out = np.empty_like(a)
    _check(_lib.lib().xa_gaussian_blur(e.handle, _ptr(a), a.shape[1], a.shape[0], sigma, _ptr(out)))
    return out


def resize_bilinear(img, new_w: int, new_h: int, engine: Engine = None) -> np.ndarray:
    a = _img(img)
    e = engine or default_engine()
    out = np.empty((new_h, new_w), np.float32)
    _check(_lib.lib().xa_resize_bilinear(e.handle, _ptr(a), a.shape[1], a.shape[0], new_w, new_h,
                                         _ptr(out)))
    return out


def antialias_tilt(img, t: float, phi: float, engine: Engine = None) -> np.ndarray:
    a = _img(img)
    e = engine or default_engine()
    out = np.empty_like(a)
    _check(_lib.lib().xa_antialias_tilt(e.handle, _ptr(a), a.shape[1], a.shape[0], t, phi,
                                        _ptr(out)))
    return out


@dataclasses.dataclass
class WarpResult:
    """xaffine::WarpResult (warp.hpp:11-16)."""
    image: np.ndarray
    tx: float
    ty: float
    forward: np.ndarray


def _warp(mode: int, img, m, a: int, engine: Engine) -> WarpResult:
    src = _img(img)
    e = engine or default_engine()
    mm = _mat(m)
    W, H = C.c_int(), C.c_int()
    tx, ty = C.c_double(), C.c_double()
    fwd = np.zeros(9, np.float64)
    _check(_lib.lib().xa_warp_frame(_ptr(mm), src.shape[1], src.shape[0], C.byref(W), C.byref(H),
                                    C.byref(tx), C.byref(ty), _ptr(fwd)))
    out = np.zeros((H.value, W.value), np.float32)
    _check(_lib.lib().xa_warp(e.handle, mode, _ptr(src), src.shape[1], src.shape[0], _ptr(mm), a,
                              _ptr(out), out.size, C.byref(W), C.byref(H), C.byref(tx),
                              C.byref(ty), _ptr(fwd)))
    return WarpResult(out, tx.value, ty.value, fwd.reshape(3, 3))


def warp_nearest(img, m, engine: Engine = None) -> WarpResult:
    return _warp(XA_NEAREST, img, m, 4, engine)


def warp_lanczos(img, m, a: int = 4, engine: Engine = None) -> WarpResult:
    return _warp(XA_LANCZOS, img, m, a, engine)


def synth_warp_case(img, h, out: str = "f32", engine: Engine = None):
    """xaffine::synth_warp_case (eval.hpp:56-60, eval.cpp:101-141): img rendered
    under the 3x3 homography h with Lanczos-4 on the device, in the warp
    module's half-pixel framing. Returns (image, composed 3x3): float32 as the
    reference returns it, or out="u8" for the lround + clamp bytes save_image
    writes (image_io.cpp:17-20). Raises EvalError for degenerate homographies."""
    if out not in ("f32", "u8"):
        raise ValueError("out must be 'f32' or 'u8'")
    src = _img(img)
    e = engine or default_engine()
    hm = _mat(h)
    ot = XA_F32 if out == "f32" else XA_U8
    W, H = C.c_int(), C.c_int()
    comp = np.zeros(9, np.float64)
    _check(_lib.lib().xa_synth_warp_case(e.handle, _ptr(src), src.shape[1], src.shape[0], _ptr(hm),
                                         ot, None, 0, C.byref(W), C.byref(H), _ptr(comp)))
    res = np.zeros((H.value, W.value), np.float32 if ot == XA_F32 else np.uint8)
    _check(_lib.lib().xa_synth_warp_case(e.handle, _ptr(src), src.shape[1], src.shape[0], _ptr(hm),
                                         ot, _ptr(res), res.size, C.byref(W), C.byref(H),
                                         _ptr(comp)))
    return res, comp.reshape(3, 3)


# ------------------------------------------------------------------ ORB

def as_keypoints(kps) -> np.ndarray:
    """Accepts a KEYPOINT structured array or an (n, 5) float array."""
    k = np.asarray(kps)
    if k.dtype == KEYPOINT:
        return np.ascontiguousarray(k)
    k = np.ascontiguousarray(k, dtype=np.float32).reshape(-1, 5)
    return k.view(KEYPOINT).reshape(-1)


def detect_oriented_corners(img, max_points: int, engine: Engine = None) -> np.ndarray:
    a = _img(img)
    e = engine or default_engine()
    cap = max(int(max_points), 0)
    out = np.zeros(max(cap, 1), KEYPOINT)
    n = C.c_int()
    _check(_lib.lib().xa_detect_oriented_corners(e.handle, _ptr(a), a.shape[1], a.shape[0],
                                                 int(max_points), _ptr(out), cap, C.byref(n)))
    return out[:n.value].copy()


def describe_binary(img, kps, engine: Engine = None) -> Tuple[np.ndarray, np.ndarray]:
    a = _img(img)
    e = engine or default_engine()
    k = as_keypoints(kps)
    n = len(k)
    ok = np.zeros(max(n, 1), KEYPOINT)
    od = np.zeros((max(n, 1), 4), np.uint64)
    m = C.c_int()
    _check(_lib.lib().xa_describe_binary(e.handle, _ptr(a), a.shape[1], a.shape[0], _ptr(k), n,
                                         _ptr(ok), _ptr(od), C.byref(m)))
    return ok[:m.value].copy(), od[:m.value].copy()


def hamming_distance(a, b) -> int:
    """features.hpp:27 / orb.cpp:176-180 (host helper, bit count of the XOR)."""
    x = np.bitwise_xor(np.asarray(a, np.uint64), np.asarray(b, np.uint64))
    return int(sum(bin(int(v)).count("1") for v in x.reshape(-1)))


def match_hamming(desc_a, desc_b, ratio: float, engine: Engine = None) -> np.ndarray:
    A = np.ascontiguousarray(np.asarray(desc_a, np.uint64).reshape(-1, 4))
    B = np.ascontiguousarray(np.asarray(desc_b, np.uint64).reshape(-1, 4))
    e = engine or default_engine()
    out = np.zeros(max(len(A), 1), MATCH)
    n = C.c_int()
    _check(_lib.lib().xa_match_hamming(e.handle, _ptr(A), len(A), _ptr(B), len(B), float(ratio),
                                       _ptr(out), C.byref(n)))
    return out[:n.value].copy()


def detect_dog_keypoints(img, max_points: int, engine: Engine = None) -> np.ndarray:
    """sift.hpp:12-13 / sift.cpp:290-358: the fine stage's DoG keypoints (N, 5)
    float32 (x, y, response, orientation, octave_scale)."""
    a = _img(img)
    h, w = a.shape
    e = engine or default_engine()
    out = np.zeros((max(max_points, 1), 5), np.float32)
    n = C.c_int()
    _check(_lib.lib().xa_detect_dog_keypoints(e.handle, _ptr(a), w, h, int(max_points), _ptr(out),
                                              len(out), C.byref(n)))
    return out[:n.value].copy()


def describe_gradient(img, kps, engine: Engine = None) -> Tuple[np.ndarray, np.ndarray]:
    """sift.hpp:18-23 / sift.cpp:360-386: (surviving keypoints (M, 5), descriptors (M, 128))."""
    a = _img(img)
    h, w = a.shape
    k = np.ascontiguousarray(np.asarray(kps, np.float32).reshape(-1, 5))
    e = engine or default_engine()
    ok = np.zeros((max(len(k), 1), 5), np.float32)
    od = np.zeros((max(len(k), 1), 128), np.float32)
    n = C.c_int()
    _check(_lib.lib().xa_describe_gradient(e.handle, _ptr(a), w, h, _ptr(k), len(k), _ptr(ok), _ptr(od),
                                           C.byref(n)))
    return ok[:n.value].copy(), od[:n.value].copy()


def match_ratio(desc_a, desc_b, ratio: float = 0.75, engine: Engine = None) -> np.ndarray:
    """sift.hpp:25-30 / sift.cpp:388-418: L2 ratio matcher over 128-float
    gradient descriptors; structured (idx_a, idx_b, distance) sorted by idx_a."""
    A = np.ascontiguousarray(np.asarray(desc_a, np.float32).reshape(-1, 128))
    B = np.ascontiguousarray(np.asarray(desc_b, np.float32).reshape(-1, 128))
    e = engine or default_engine()
    out = np.zeros(max(len(A), 1), MATCH)
    n = C.c_int()
    _check(_lib.lib().xa_match_ratio(e.handle, _ptr(A), len(A), _ptr(B), len(B), float(ratio),
                                     _ptr(out), C.byref(n)))
    return out[:n.value].copy()


# ------------------------------------------------------------------ fine stage (§8f)

def filter_to_content(kps, back, src_w: int, src_h: int, margin: float) -> np.ndarray:
    """pipeline.cpp:28-40: keep keypoints whose back-mapped position lies at
    least `margin` inside the source (host double arithmetic)."""
    k = np.asarray(kps, np.float32).reshape(-1, 5)
    b = np.asarray(back, np.float64).reshape(3, 3)
    keep = []
    for i, (x, y) in enumerate(k[:, :2].astype(np.float64)):
        sx, sy = map_point(b, float(x), float(y))
        keep.append(margin <= sx <= src_w - 1 - margin and margin <= sy <= src_h - 1 - margin)
    return k[np.asarray(keep, bool)] if len(k) else k


def fine_features(img, cap: int, engine: Engine = None) -> Tuple[np.ndarray, np.ndarray]:
    """pipeline.cpp:47-51: SIFT keypoints + gradient descriptors (device)."""
    return describe_gradient(img, detect_dog_keypoints(img, cap, engine=engine), engine=engine)


@dataclasses.dataclass
class ReferenceDecision:
    """xaffine::ReferenceDecision (pipeline.hpp:32-37)."""
    reference: int = 1
    f_forward: float = 0.0
    f_backward: float = 0.0
    segment_count: int = 0


def scaling_coefficient(kps_a, kps_b, matches) -> Tuple[float, int]:
    """pipeline.cpp:71-103 (Eq. 1): weighted sum of matched-segment length
    differences over every fourth rank of the distance-sorted matches. The
    reference takes the keypoint differences and hypot in float precision and
    the weight from a float distance sum; replayed here with float32 numpy."""
    n = len(matches)
    if n < 2:
        raise PipelineError("insufficient matches for scaling estimation")
    ka = np.asarray(kps_a, np.float32).reshape(-1, 5)
    kb = np.asarray(kps_b, np.float32).reshape(-1, 5)
    ia, ib = np.asarray(matches["idx_a"]), np.asarray(matches["idx_b"])
    if np.any(ia < 0) or np.any(ia >= len(ka)) or np.any(ib < 0) or np.any(ib >= len(kb)):
        raise PipelineError("match indices out of range")
    order = np.lexsort((ia, np.asarray(matches["distance"], np.float32)))
    ranked = np.asarray(matches)[order]
    f, seg = 0.0, 0
    for i in range(0, n):
        if 4 * i + 1 >= n:
            break
        m0, m1 = ranked[4 * i], ranked[4 * i + 1]
        a0, a1 = ka[m0["idx_a"]], ka[m1["idx_a"]]
        b0, b1 = kb[m0["idx_b"]], kb[m1["idx_b"]]
        dis_a = float(np.hypot(np.float32(a0[0] - a1[0]), np.float32(a0[1] - a1[1])))
        dis_b = float(np.hypot(np.float32(b0[0] - b1[0]), np.float32(b0[1] - b1[1])))
        w = max(0.0, 1.0 - float(np.float32(m0["distance"]) + np.float32(m1["distance"])) / 1000.0)
        f += (dis_a - dis_b) * w
        seg += 1
    return f, seg


def select_reference(img1, img2, cap: int = 2000, engine: Engine = None) -> ReferenceDecision:
    """pipeline.cpp:105-120: SIFT on both images, ratio-0.75 matches both ways,
    the larger scaling coefficient picks the reference image."""
    k1, d1 = fine_features(img1, cap, engine)
    k2, d2 = fine_features(img2, cap, engine)
    m12, m21 = match_ratio(d1, d2, 0.75, engine), match_ratio(d2, d1, 0.75, engine)
    d = ReferenceDecision()
    if len(m12) < 2 or len(m21) < 2:
        a1 = np.asarray(img1).shape[0] * np.asarray(img1).shape[1]
        a2 = np.asarray(img2).shape[0] * np.asarray(img2).shape[1]
        d.reference = 2 if a2 > a1 else 1
        return d
    d.f_forward, d.segment_count = scaling_coefficient(k1, k2, m12)
    d.f_backward, _ = scaling_coefficient(k2, k1, m21)
    d.reference = 1 if d.f_forward >= d.f_backward else 2
    return d


def fine_correspondences(ref, target, params: "AffineParams", max_points: int = 2000,
                         ratio: float = 0.75, lanczos_a: int = 4, engine: Engine = None):
    """fine_match (pipeline.cpp:154-190) up to the RANSAC screen, which stays on
    the host CPU (Eigen): simulate the view at the coarse pose,
    SIFT on the view (content-filtered) and on the target, L2 ratio matches,
    correspondences mapped back to the reference frame. Returns
    ((N, 5) float64 [x_ref, y_ref, x_tgt, y_tgt, distance], forward matrix)."""
    filt = antialias_tilt(ref, params.tilt, params.phi, engine=engine)
    w = warp_lanczos(filt, simulation_from_params(params), lanczos_a, engine=engine)
    back = invert(w.forward)
    kps = detect_dog_keypoints(w.image, max_points, engine=engine)
    kps = filter_to_content(kps, back, np.asarray(ref).shape[1], np.asarray(ref).shape[0], float(lanczos_a))
    wk, wd = describe_gradient(w.image, kps, engine=engine)
    tk, td = fine_features(target, max_points, engine)
    m = match_ratio(wd, td, ratio, engine)
    if len(m) < 4:
        raise PipelineError("fine: insufficient matches")
    out = np.zeros((len(m), 5), np.float64)
    for i, r in enumerate(m):
        x1, y1 = float(wk[r["idx_a"], 0]), float(wk[r["idx_a"], 1])
        out[i, 0], out[i, 1] = map_point(back, x1, y1)
        out[i, 2], out[i, 3] = float(tk[r["idx_b"], 0]), float(tk[r["idx_b"], 1])
        out[i, 4] = float(r["distance"])
    return out, w.forward


def asift_correspondences(img1, img2, grid: ParamGrid, max_points: int = 1000, ratio: float = 0.75,
                          lanczos_a: int = 4, engine: Engine = None) -> np.ndarray:
    """asift_baseline (pipeline.cpp:298-343) up to the RANSAC screen: both
    images simulated at every grid entry (scale 1), SIFT per view, L2 ratio
    matching of every view pair, 2-px duplicate suppression in pair order.
    Returns (N, 5) float64 [x1, y1, x2, y2, distance] (Correspondence)."""
    a, b = _img(img1), _img(img2)
    e = engine or default_engine()
    g = _params_array(grid.entries)
    cap = 1 << 16
    while True:
        out = np.zeros((cap, 5), np.float64)
        n = C.c_int()
        rc = _lib.lib().xa_asift_correspondences(
            e.handle, _ptr(a), a.shape[1], a.shape[0], _ptr(b), b.shape[1], b.shape[0], g,
            len(grid.entries), max_points, float(ratio), lanczos_a, _ptr(out), cap, C.byref(n))
        if rc == _lib.XA_ECAPACITY and n.value > cap:
            cap = n.value
            continue
        _check(rc)
        return out[:n.value].copy()


# ------------------------------------------------------------------ pipeline

@dataclasses.dataclass
class CoarseResult:
    """xaffine::CoarseResult (pipeline.hpp:39-43) plus per-entry described keypoints."""
    best_params: AffineParams
    best_count: int
    per_entry_counts: List[Tuple[AffineParams, int]]
    per_entry_keypoints: List[int] = dataclasses.field(default_factory=list)
    best_index: int = 0


def coarse_search(ref, target, grid: ParamGrid, max_points: int = 1000, ratio: float = 0.75,
                  warp_mode: str = "nearest", engine: Engine = None) -> CoarseResult:
    """Batched coarse_search (pipeline.cpp:122-152). ref/target: uint8 or float32 images
    (both the same type). warp_mode "nearest" is the reference's coarse resampler;
    "lanczos" is the north-star variant. Views are quantised to uint8 before ORB."""
    entries = grid.entries if isinstance(grid, ParamGrid) else list(grid)
    if not entries:
        raise PipelineError("coarse: empty parameter grid")
    r = np.asarray(ref)
    t = np.asarray(target)
    if r.dtype == np.uint8 and t.dtype == np.uint8:
        ptype = XA_U8
        r = np.ascontiguousarray(r)
        t = np.ascontiguousarray(t)
    else:
        ptype = XA_F32
        r = _img(r)
        t = _img(t)
    e = engine or default_engine()
    params = _params_array(entries)
    n = len(entries)
    counts = np.zeros(n, np.int32)
    kpc = np.zeros(n, np.int32)
    best = C.c_int32()
    mode = XA_NEAREST if warp_mode == "nearest" else XA_LANCZOS
    _check(_lib.lib().xa_coarse_search(e.handle, ptype, _ptr(r), r.shape[1], r.shape[0], _ptr(t),
                                       t.shape[1], t.shape[0], params, n, int(max_points),
                                       float(ratio), mode, _ptr(counts), _ptr(kpc), C.byref(best)))
    ents = [p if isinstance(p, AffineParams) else AffineParams(*p) for p in entries]
    bi = int(best.value)
    return CoarseResult(ents[bi], int(counts[bi]), list(zip(ents, counts.tolist())),
                        kpc.tolist(), bi)


def coarse_search_batch(refs, targets, grid: ParamGrid, max_points: int = 1000, ratio: float = 0.75,
                        warp_mode: str = "nearest", engine: Engine = None) -> List[CoarseResult]:
    """coarse_search (pipeline.cpp:122-152) over many image pairs in one batched
    device call (BASELINE config 5). All reference images share one size and all
    targets another; uint8 or float32 (one type for all)."""
    entries = grid.entries if isinstance(grid, ParamGrid) else list(grid)
    if not entries:
        raise PipelineError("coarse: empty parameter grid")
    refs, targets = [np.asarray(r) for r in refs], [np.asarray(t) for t in targets]
    if len(refs) != len(targets) or not refs:
        raise ValueError("coarse_search_batch: need the same number (>0) of references and targets")
    if all(r.dtype == np.uint8 for r in refs + targets):
        ptype = XA_U8
        refs = [np.ascontiguousarray(r) for r in refs]
        targets = [np.ascontiguousarray(t) for t in targets]
    else:
        ptype = XA_F32
        refs = [_img(r) for r in refs]
        targets = [_img(t) for t in targets]
    if len({r.shape for r in refs}) != 1 or len({t.shape for t in targets}) != 1:
        raise ValueError("coarse_search_batch: references (and targets) must share one size")
    e = engine or default_engine()
    params = _params_array(entries)
    n, P = len(entries), len(refs)
    counts = np.zeros((P, n), np.int32)
    kpc = np.zeros((P, n), np.int32)
    best = np.zeros(P, np.int32)
    R = (C.c_void_p * P)(*[_ptr(r) for r in refs])
    T = (C.c_void_p * P)(*[_ptr(t) for t in targets])
    mode = XA_NEAREST if warp_mode == "nearest" else XA_LANCZOS
    _check(_lib.lib().xa_coarse_search_batch(
        e.handle, ptype, R, refs[0].shape[1], refs[0].shape[0], T, targets[0].shape[1],
        targets[0].shape[0], P, params, n, int(max_points), float(ratio), mode, _ptr(counts),
        _ptr(kpc), _ptr(best)))
    ents = [p if isinstance(p, AffineParams) else AffineParams(*p) for p in entries]
    out = []
    for p in range(P):
        bi = int(best[p])
        out.append(CoarseResult(ents[bi], int(counts[p, bi]), list(zip(ents, counts[p].tolist())),
                                kpc[p].tolist(), bi))
    return out


def coarse_search_multi(refs, targets, grid: ParamGrid, max_points: int = 1000, ratio: float = 0.75,
                        warp_mode: str = "nearest", engines: Sequence[Engine] = None) -> List[CoarseResult]:
    """coarse_search_batch sharded over several engines (one per GPU) in this
    process: contiguous blocks of pairs, one host thread per engine
    (xa_coarse_search_multi)."""
    return _multi_call(refs, targets, grid, max_points, ratio, warp_mode, engines=engines)


def coarse_search_nccl(refs, targets, grid: ParamGrid, comm: int, rank: int, world: int,
                       max_points: int = 1000, ratio: float = 0.75, warp_mode: str = "nearest",
                       engine: Engine = None) -> List[CoarseResult]:
    """One rank of a multi-process run: this rank's block of pairs on its GPU,
    then every rank's results all-gathered over the NCCL communicator `comm`
    (an ncclComm_t address, e.g. from nccl_comm_init) -- xa_coarse_search_nccl."""
    return _multi_call(refs, targets, grid, max_points, ratio, warp_mode, engine=engine, comm=comm,
                       rank=rank, world=world)


def nccl_unique_id() -> bytes:
    buf = (C.c_char * 128)()
    _check_multi(_lib.lib().xa_nccl_unique_id(buf, 128))
    return bytes(buf)


def nccl_comm_init(uid: bytes, rank: int, world: int, device: int = 0) -> int:
    comm = C.c_void_p()
    buf = (C.c_char * 128).from_buffer_copy(uid)
    _check_multi(_lib.lib().xa_nccl_comm_init(C.byref(comm), world, buf, rank, device))
    return comm.value


def nccl_comm_destroy(comm: int) -> None:
    _lib.lib().xa_nccl_comm_destroy(C.c_void_p(comm))


def _check_multi(rc: int) -> None:
    if rc != _lib.XA_OK:
        raise XaError(rc, _lib.lib().xa_multi_last_error().decode())


def _multi_call(refs, targets, grid, max_points, ratio, warp_mode, engines=None, engine=None, comm=None,
                rank=0, world=1):
    entries = grid.entries if isinstance(grid, ParamGrid) else list(grid)
    if not entries:
        raise PipelineError("coarse: empty parameter grid")
    refs, targets = [np.asarray(r) for r in refs], [np.asarray(t) for t in targets]
    if all(r.dtype == np.uint8 for r in refs + targets):
        ptype = XA_U8
        refs = [np.ascontiguousarray(r) for r in refs]
        targets = [np.ascontiguousarray(t) for t in targets]
    else:
        ptype = XA_F32
        refs = [_img(r) for r in refs]
        targets = [_img(t) for t in targets]
    if len({r.shape for r in refs}) != 1 or len({t.shape for t in targets}) != 1:
        raise ValueError("coarse_search: references (and targets) must share one size")
    params = _params_array(entries)
    n, P = len(entries), len(refs)
    counts = np.zeros((P, n), np.int32)
    kpc = np.zeros((P, n), np.int32)
    best = np.zeros(P, np.int32)
    R = (C.c_void_p * P)(*[_ptr(r) for r in refs])
    T = (C.c_void_p * P)(*[_ptr(t) for t in targets])
    mode = XA_NEAREST if warp_mode == "nearest" else XA_LANCZOS
    L = _lib.lib()
    args = (ptype, R, refs[0].shape[1], refs[0].shape[0], T, targets[0].shape[1], targets[0].shape[0], P,
            params, n, int(max_points), float(ratio), mode, _ptr(counts), _ptr(kpc), _ptr(best))
    if comm is None:
        engines = list(engines or [default_engine()])
        E = (C.c_void_p * len(engines))(*[e.handle for e in engines])
        _check_multi(L.xa_coarse_search_multi(E, len(engines), *args))
    else:
        e = engine or default_engine()
        _check_multi(L.xa_coarse_search_nccl(e.handle, C.c_void_p(comm), rank, world, *args))
    ents = [p if isinstance(p, AffineParams) else AffineParams(*p) for p in entries]
    return [CoarseResult(ents[int(best[p])], int(counts[p, int(best[p])]),
                         list(zip(ents, counts[p].tolist())), kpc[p].tolist(), int(best[p]))
            for p in range(P)]


# ------------------------------------------------------------------ image I/O

def load_image(path) -> np.ndarray:
    """load_image (image_io.hpp:14-16): PGM/PPM (P2, P3, P5, P6) or PNG as a float32
    (h, w) grayscale raster; colour -> (float)(0.299 R + 0.587 G + 0.114 B)."""
    p = str(path).encode()
    w, h = C.c_int(), C.c_int()
    _check(_lib.lib().xa_load_image(p, None, 0, C.byref(w), C.byref(h)))
    out = np.zeros((h.value, w.value), np.float32)
    _check(_lib.lib().xa_load_image(p, _ptr(out), out.size, C.byref(w), C.byref(h)))
    return out


def save_image(img, path) -> None:
    """save_image (image_io.hpp:18-19): 8-bit grayscale .pgm (P5) or .png, each
    pixel lround + clamp to [0, 255] (image_io.cpp:18-21)."""
    a = _img(img)
    _check(_lib.lib().xa_save_image(_ptr(a), a.shape[1], a.shape[0], str(path).encode()))


def save_png_rgb(rgb, path) -> None:
    """save_png_rgb (image_io.hpp:21-22): (h, w, 3) uint8 -> 8-bit RGB PNG."""
    a = np.ascontiguousarray(np.asarray(rgb, np.uint8))
    if a.ndim != 3 or a.shape[2] != 3:
        raise ValueError("save_png_rgb: expected an (h, w, 3) uint8 image")
    _check(_lib.lib().xa_save_png_rgb(_ptr(a), a.shape[1], a.shape[0], str(path).encode()))


def quantize(img) -> np.ndarray:
    """The uint8 quantisation of save_image (lround + clamp, image_io.cpp:18-21)."""
    a = np.ascontiguousarray(np.asarray(img, np.float32))
    out = np.zeros(a.shape, np.uint8)
    _check(_lib.lib().xa_quantize(_ptr(a), a.size, _ptr(out)))
    return out


# ------------------------------------------------------------------ geometric verification

def _points(pts) -> np.ndarray:
    """PointPair list (x1, y1, x2, y2) as a contiguous (n, 4) float64 array."""
    a = np.asarray(pts, np.float64)
    return np.ascontiguousarray(a.reshape(-1, 4)) if a.size else np.zeros((0, 4))


def fit_homography_dlt(pts) -> np.ndarray:
    """fit_homography_dlt (homography.hpp:27-29): normalised DLT, h22 = 1."""
    a = _points(pts)
    h = np.zeros(9)
    _check(_lib.lib().xa_fit_homography_dlt(_ptr(a), len(a), _ptr(h)))
    return h.reshape(3, 3)


def estimate_homography_ransac(pts, threshold: float = 3.0, max_iters: int = 2000,
                               confidence: float = 0.995, seed: int = 42):
    """estimate_homography_ransac (homography.hpp:35-39) with RansacConfig's
    defaults -> (homography (3, 3), inlier indices)."""
    a = _points(pts)
    h = np.zeros(9)
    inl = np.zeros(max(len(a), 1), np.int32)
    n = C.c_int()
    _check(_lib.lib().xa_estimate_homography_ransac(_ptr(a), len(a), float(threshold), int(max_iters),
                                                    float(confidence), int(seed), _ptr(h), _ptr(inl),
                                                    len(inl), C.byref(n)))
    return h.reshape(3, 3), inl[:n.value].copy()
