"""ctypes face of the CPU checkers — TEST INFRASTRUCTURE ONLY.

`Oracle("port")` loads oracle/libxaoracle.so (the C restatement, always built by
`make -C oracle`); `Oracle("reference")` loads oracle/_ref/libxaref.so (the
reference library compiled from /root/reference, present only where it was
built). Both expose the same `orc_*` C interface (oracle/xa_oracle.h), so every
method here returns identical structures for both. Only tests/, smoke() and
bench.py's cpu_baseline / --impl reference legs may import this module.
"""
from __future__ import annotations

import ctypes as C
import os
import pathlib

import numpy as np

HERE = pathlib.Path(__file__).resolve().parent
PATHS = {
    "port": HERE / "libxaoracle.so",
    "reference": HERE / "_ref" / "libxaref.so",
    "reference_popcnt": HERE / "_ref" / "libxaref_popcnt.so",
}

_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_pp = C.POINTER(C.c_void_p)


def available(kind: str) -> bool:
    return PATHS[kind].exists()


class OracleError(RuntimeError):
    pass


class Oracle:
    def __init__(self, kind: str = "port"):
        path = PATHS[kind]
        if not path.exists():
            raise FileNotFoundError(f"{path} not built (make -C oracle)")
        self.kind = kind
        L = self.lib = C.CDLL(str(path))
        L.orc_last_error.restype = C.c_char_p
        L.orc_pattern_checksum.restype = C.c_uint64
        L.orc_lanczos_kernel.restype = C.c_double
        L.orc_lanczos_kernel.argtypes = [C.c_double, C.c_int]
        L.orc_sample_lanczos.restype = C.c_double
        L.orc_sample_lanczos.argtypes = [_f32p, C.c_int, C.c_int, C.c_double, C.c_double, C.c_int]
        L.orc_free.argtypes = [C.c_void_p]

    # ------------------------------------------------------------ helpers
    def _ok(self, rc):
        if rc != 0:
            raise OracleError(self.lib.orc_last_error().decode())

    def _take(self, ptr, n, dtype):
        """Copy n elements out of a library-malloc'd buffer and free it."""
        try:
            if n == 0:
                return np.zeros(0, dtype)
            buf = (C.c_char * (n * np.dtype(dtype).itemsize)).from_address(ptr.value)
            return np.frombuffer(bytes(buf), dtype=dtype).copy()
        finally:
            self.lib.orc_free(ptr)

    @staticmethod
    def _img(img):
        a = np.ascontiguousarray(img, dtype=np.float32)
        assert a.ndim == 2
        return a, a.shape[1], a.shape[0]

    # ------------------------------------------------------------ pattern
    def pattern_checksum(self) -> int:
        return int(self.lib.orc_pattern_checksum())

    def pattern(self) -> np.ndarray:
        buf = (C.c_int8 * 1024)()
        self.lib.orc_pattern(buf)
        return np.frombuffer(bytes(buf), np.int8).reshape(256, 4).copy()

    # ------------------------------------------------------------ images
    def make_texture(self, w, h, seed=7):
        out = np.zeros((h, w), np.float32)
        self._ok(self.lib.orc_make_texture(C.c_int(w), C.c_int(h), C.c_uint64(seed),
                                           out.ctypes.data_as(C.c_void_p)))
        return out

    def make_checkerboard(self, w, h, cell):
        out = np.zeros((h, w), np.float32)
        self._ok(self.lib.orc_make_checkerboard(w, h, cell, out.ctypes.data_as(C.c_void_p)))
        return out

    def gaussian_blur(self, img, sigma):
        a, w, h = self._img(img)
        out = np.zeros_like(a)
        self._ok(self.lib.orc_gaussian_blur(a.ctypes.data_as(C.c_void_p), w, h, C.c_double(sigma),
                                            out.ctypes.data_as(C.c_void_p)))
        return out

    def resize_bilinear(self, img, nw, nh):
        a, w, h = self._img(img)
        out = np.zeros((nh, nw), np.float32)
        self._ok(self.lib.orc_resize_bilinear(a.ctypes.data_as(C.c_void_p), w, h, nw, nh,
                                              out.ctypes.data_as(C.c_void_p)))
        return out

    def antialias_tilt(self, img, t, phi):
        a, w, h = self._img(img)
        out = np.zeros_like(a)
        self._ok(self.lib.orc_antialias_tilt(a.ctypes.data_as(C.c_void_p), w, h, C.c_double(t),
                                             C.c_double(phi), out.ctypes.data_as(C.c_void_p)))
        return out

    def lanczos_kernel(self, x, a=4):
        return self.lib.orc_lanczos_kernel(x, a)

    def sample_lanczos(self, img, x, y, a=4):
        arr, w, h = self._img(img)
        return self.lib.orc_sample_lanczos(arr, w, h, x, y, a)

    def warp(self, img, m, mode="nearest", a=4):
        """Returns (image, tx, ty, forward 3x3)."""
        arr, w, h = self._img(img)
        m = np.ascontiguousarray(np.asarray(m, np.float64).reshape(9))
        out = C.c_void_p()
        W, H = C.c_int(), C.c_int()
        tx, ty = C.c_double(), C.c_double()
        fwd = np.zeros(9, np.float64)
        self._ok(self.lib.orc_warp(0 if mode == "nearest" else 1, arr.ctypes.data_as(C.c_void_p),
                                   w, h, m.ctypes.data_as(C.c_void_p), a, C.byref(out),
                                   C.byref(W), C.byref(H), C.byref(tx), C.byref(ty),
                                   fwd.ctypes.data_as(C.c_void_p)))
        im = self._take(out, W.value * H.value, np.float32).reshape(H.value, W.value)
        return im, tx.value, ty.value, fwd.reshape(3, 3)

    def synth_warp_case(self, img, h):
        """eval.cpp:101-141 -> (float32 image, composed 3x3)."""
        arr, w, hh = self._img(img)
        hm = np.ascontiguousarray(np.asarray(h, np.float64).reshape(9))
        out = C.c_void_p()
        W, H = C.c_int(), C.c_int()
        comp = np.zeros(9, np.float64)
        self._ok(self.lib.orc_synth_warp_case(arr.ctypes.data_as(C.c_void_p), w, hh,
                                              hm.ctypes.data_as(C.c_void_p), C.byref(out),
                                              C.byref(W), C.byref(H),
                                              comp.ctypes.data_as(C.c_void_p)))
        im = self._take(out, W.value * H.value, np.float32).reshape(H.value, W.value)
        return im, comp.reshape(3, 3)

    def warp_nearest(self, img, m):
        return self.warp(img, m, "nearest")

    def warp_lanczos(self, img, m, a=4):
        return self.warp(img, m, "lanczos", a)

    # ------------------------------------------------------------ ORB
    def detect(self, img, max_points):
        arr, w, h = self._img(img)
        p, n = C.c_void_p(), C.c_int()
        self._ok(self.lib.orc_detect(arr.ctypes.data_as(C.c_void_p), w, h, max_points,
                                     C.byref(p), C.byref(n)))
        return self._take(p, 5 * n.value, np.float32).reshape(n.value, 5)

    def detect_dog(self, img, max_points):
        """detect_dog_keypoints (sift.cpp:290-358) -> (n, 5) float32."""
        arr, w, h = self._img(img)
        p, n = C.c_void_p(), C.c_int()
        self._ok(self.lib.orc_detect_dog(arr.ctypes.data_as(C.c_void_p), w, h, max_points,
                                         C.byref(p), C.byref(n)))
        return self._take(p, 5 * n.value, np.float32).reshape(n.value, 5)

    def describe_gradient(self, img, kps):
        """describe_gradient (sift.cpp:360-386) -> ((m, 5) keypoints, (m, 128) float32)."""
        arr, w, h = self._img(img)
        k = np.ascontiguousarray(np.asarray(kps, np.float32).reshape(-1, 5))
        pk, pd, n = C.c_void_p(), C.c_void_p(), C.c_int()
        self._ok(self.lib.orc_describe_gradient(arr.ctypes.data_as(C.c_void_p), w, h,
                                                k.ctypes.data_as(C.c_void_p), len(k), C.byref(pk),
                                                C.byref(pd), C.byref(n)))
        m = n.value
        return (self._take(pk, 5 * m, np.float32).reshape(m, 5),
                self._take(pd, 128 * m, np.float32).reshape(m, 128))

    def describe(self, img, kps):
        arr, w, h = self._img(img)
        k = np.ascontiguousarray(np.asarray(kps, np.float32).reshape(-1, 5))
        pk, pd, n = C.c_void_p(), C.c_void_p(), C.c_int()
        self._ok(self.lib.orc_describe(arr.ctypes.data_as(C.c_void_p), w, h,
                                       k.ctypes.data_as(C.c_void_p), len(k), C.byref(pk),
                                       C.byref(pd), C.byref(n)))
        kk = self._take(pk, 5 * n.value, np.float32).reshape(n.value, 5)
        dd = self._take(pd, 4 * n.value, np.uint64).reshape(n.value, 4)
        return kk, dd

    def match(self, a, b, ratio):
        a = np.ascontiguousarray(np.asarray(a, np.uint64).reshape(-1, 4))
        b = np.ascontiguousarray(np.asarray(b, np.uint64).reshape(-1, 4))
        p, n = C.c_void_p(), C.c_int()
        self._ok(self.lib.orc_match(a.ctypes.data_as(C.c_void_p), len(a),
                                    b.ctypes.data_as(C.c_void_p), len(b), C.c_double(ratio),
                                    C.byref(p), C.byref(n)))
        return self._take(p, 3 * n.value, np.int32).reshape(n.value, 3)

    def match_ratio(self, a, b, ratio):
        """match_ratio (sift.cpp:388-418) -> structured (idx_a, idx_b, distance)."""
        a = np.ascontiguousarray(np.asarray(a, np.float32).reshape(-1, 128))
        b = np.ascontiguousarray(np.asarray(b, np.float32).reshape(-1, 128))
        p, n = C.c_void_p(), C.c_int()
        self._ok(self.lib.orc_match_ratio(a.ctypes.data_as(C.c_void_p), len(a),
                                          b.ctypes.data_as(C.c_void_p), len(b), C.c_double(ratio),
                                          C.byref(p), C.byref(n)))
        raw = self._take(p, 3 * n.value, np.int32).reshape(n.value, 3)
        out = np.zeros(n.value, dtype=[("idx_a", np.int32), ("idx_b", np.int32), ("distance", np.float32)])
        out["idx_a"], out["idx_b"] = raw[:, 0], raw[:, 1]
        out["distance"] = raw[:, 2].copy().view(np.float32)
        return out

    def scaling_coefficient(self, kps_a, kps_b, matches):
        """scaling_coefficient (pipeline.cpp:70-101) -> (f, segments)."""
        ka = np.ascontiguousarray(np.asarray(kps_a, np.float32).reshape(-1, 5))
        kb = np.ascontiguousarray(np.asarray(kps_b, np.float32).reshape(-1, 5))
        m = np.zeros((len(matches), 3), np.int32)
        m[:, 0], m[:, 1] = matches["idx_a"], matches["idx_b"]
        m[:, 2] = np.asarray(matches["distance"], np.float32).view(np.int32)
        f, seg = C.c_double(), C.c_int()
        self._ok(self.lib.orc_scaling_coefficient(
            ka.ctypes.data_as(C.c_void_p), len(ka), kb.ctypes.data_as(C.c_void_p), len(kb),
            m.ctypes.data_as(C.c_void_p), len(m), C.byref(f), C.byref(seg)))
        return f.value, seg.value

    def select_reference(self, img1, img2, cap=1000):
        """select_reference (pipeline.cpp:103-120) -> (reference, f_fwd, f_bwd, segments)."""
        a, w1, h1 = self._img(img1)
        b, w2, h2 = self._img(img2)
        r, ff, fb, seg = C.c_int(), C.c_double(), C.c_double(), C.c_int()
        self._ok(self.lib.orc_select_reference(
            a.ctypes.data_as(C.c_void_p), w1, h1, b.ctypes.data_as(C.c_void_p), w2, h2, cap,
            C.byref(r), C.byref(ff), C.byref(fb), C.byref(seg)))
        return r.value, ff.value, fb.value, seg.value

    def asift_correspondences(self, img1, img2, grid, cap=1000, ratio=0.75, a=4):
        """asift_baseline (pipeline.cpp:298-343) up to RANSAC -> (N, 5) float64."""
        x, w1, h1 = self._img(img1)
        y, w2, h2 = self._img(img2)
        g = np.ascontiguousarray(np.asarray(grid, np.float64).reshape(-1, 6))
        p, n = C.c_void_p(), C.c_int()
        self._ok(self.lib.orc_asift_correspondences(
            x.ctypes.data_as(C.c_void_p), w1, h1, y.ctypes.data_as(C.c_void_p), w2, h2,
            g.ctypes.data_as(C.c_void_p), len(g), cap, C.c_double(ratio), a, C.byref(p), C.byref(n)))
        return self._take(p, 5 * n.value, np.float64).reshape(n.value, 5)

    # ------------------------------------------------------------ geometry
    def build_grid(self, a=2 ** 0.5, n=5, b_deg=72.0, delta_s=0.5):
        p, cnt = C.c_void_p(), C.c_int()
        self._ok(self.lib.orc_build_grid(C.c_double(a), n, C.c_double(b_deg), C.c_double(delta_s),
                                         C.byref(p), C.byref(cnt)))
        return self._take(p, 6 * cnt.value, np.float64).reshape(cnt.value, 6)

    def _mat_fn(self, fn, x):
        x = np.ascontiguousarray(np.asarray(x, np.float64).reshape(-1))
        out = np.zeros(9, np.float64)
        self._ok(fn(x.ctypes.data_as(C.c_void_p), out.ctypes.data_as(C.c_void_p)))
        return out.reshape(3, 3)

    def simulation_from_params(self, p):
        return self._mat_fn(self.lib.orc_simulation_from_params, p)

    def affine_from_params(self, p):
        return self._mat_fn(self.lib.orc_affine_from_params, p)

    def invert(self, m):
        return self._mat_fn(self.lib.orc_invert, m)

    def filter_to_content(self, kps, back, src_w, src_h, margin=5.0):
        k = np.ascontiguousarray(np.asarray(kps, np.float32).reshape(-1, 5))
        b = np.ascontiguousarray(np.asarray(back, np.float64).reshape(9))
        p, n = C.c_void_p(), C.c_int()
        self._ok(self.lib.orc_filter_to_content(k.ctypes.data_as(C.c_void_p), len(k),
                                                b.ctypes.data_as(C.c_void_p), src_w, src_h,
                                                C.c_double(margin), C.byref(p), C.byref(n)))
        return self._take(p, 5 * n.value, np.float32).reshape(n.value, 5)

    def coarse_search(self, ref, target, grid, max_points=1000, ratio=0.75, mode="nearest",
                      threads=None):
        """Returns (counts[n], kp_counts[n] (-1 if unknown), best_index)."""
        r, w, h = self._img(ref)
        t, tw, th = self._img(target)
        g = np.ascontiguousarray(np.asarray(grid, np.float64).reshape(-1, 6))
        n = len(g)
        counts = np.zeros(n, np.int32)
        kpc = np.zeros(n, np.int32)
        best = C.c_int()
        old = os.environ.get("XAFFINE_THREADS")
        if threads is not None:
            os.environ["XAFFINE_THREADS"] = str(threads)
            if hasattr(self.lib, "orc_set_threads"):
                self.lib.orc_set_threads(int(threads))
        try:
            self._ok(self.lib.orc_coarse_search(
                r.ctypes.data_as(C.c_void_p), w, h, t.ctypes.data_as(C.c_void_p), tw, th,
                g.ctypes.data_as(C.c_void_p), n, max_points, C.c_double(ratio),
                {"nearest": 0, "lanczos": 1, "nearest_u8": 2, "lanczos_u8": 3}[mode],
                counts.ctypes.data_as(C.c_void_p),
                kpc.ctypes.data_as(C.c_void_p), C.byref(best)))
        finally:
            if threads is not None:
                if old is None:
                    os.environ.pop("XAFFINE_THREADS", None)
                else:
                    os.environ["XAFFINE_THREADS"] = old
        return counts, kpc, best.value

    # ------------------------------------------------------------ probes (port only)
    def detect_candidates(self, img, thr):
        arr, w, h = self._img(img)
        pxy, ps, n = C.c_void_p(), C.c_void_p(), C.c_int()
        self._ok(self.lib.orc_detect_candidates(arr.ctypes.data_as(C.c_void_p), w, h,
                                                C.c_float(thr), C.byref(pxy), C.byref(ps),
                                                C.byref(n)))
        xyl = self._take(pxy, 3 * n.value, np.int32).reshape(n.value, 3)
        sc = self._take(ps, n.value, np.float32)
        return xyl, sc

    def corner_measures(self, level_img, xy):
        arr, w, h = self._img(level_img)
        xy = np.ascontiguousarray(np.asarray(xy, np.int32).reshape(-1, 2))
        resp = np.zeros(len(xy), np.float32)
        ori = np.zeros(len(xy), np.float32)
        self._ok(self.lib.orc_corner_measures(arr.ctypes.data_as(C.c_void_p), w, h,
                                              xy.ctypes.data_as(C.c_void_p), len(xy),
                                              resp.ctypes.data_as(C.c_void_p),
                                              ori.ctypes.data_as(C.c_void_p)))
        return resp, ori
