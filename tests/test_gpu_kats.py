"""The reference's remaining property tests restated against the device path
(proj/tests/test_features_binary.cpp, test_warp.cpp, test_geometry.cpp):
rotation repeatability, rotated-descriptor robustness, Hamming metric axioms,
ratio nesting, simulation determinant, Lanczos round trip."""
import math

import numpy as np
import pytest

from _mt64 import random_descriptors

pytestmark = pytest.mark.gpu


def _rot(a):
    c, s = math.cos(a), math.sin(a)  # AffineMatrix::rotation (geometry.cpp:18-26)
    return np.array([[c, -s, 0.0], [s, c, 0.0], [0.0, 0.0, 1.0]])


def _kps(k):
    return np.asarray(k).view(np.float32).reshape(-1, 5)


def test_rotation_90_repeatability(xa, port):
    # test_features_binary.cpp:103-119
    img = port.make_texture(200, 200, 33)
    rot = xa.warp_nearest(img, _rot(math.pi / 2))
    k1 = _kps(xa.detect_oriented_corners(img, 500))
    k2 = _kps(xa.detect_oriented_corners(rot.image, 500))
    assert len(k1) > 100
    found = 0
    for x, y in k1[:, :2]:
        rx, ry = xa.map_point(rot.forward, float(x), float(y))
        if np.any(np.hypot(k2[:, 0] - rx, k2[:, 1] - ry) <= 2.0):
            found += 1
    assert found >= len(k1) * 8 // 10


def test_descriptors_robust_to_30deg_rotation(xa, port):
    # test_features_binary.cpp:154-188
    img = port.make_checkerboard(256, 256, 32)
    ang = math.pi / 6
    rot = xa.warp_lanczos(img, _rot(ang), 4)
    k1, d1 = xa.describe_binary(img, xa.detect_oriented_corners(img, 300))
    k1 = _kps(k1).copy()
    assert len(d1) > 50
    mapped = k1.copy()
    for i, (x, y) in enumerate(k1[:, :2]):
        rx, ry = xa.map_point(rot.forward, float(x), float(y))
        mapped[i, 0], mapped[i, 1] = np.float32(rx), np.float32(ry)
        mapped[i, 3] = np.float32(float(k1[i, 3]) + ang)
    k2, d2 = xa.describe_binary(rot.image, mapped)
    k2 = _kps(k2)
    assert len(d2) > 30
    good = total = cursor = 0
    for j in range(len(k2)):
        while cursor < len(mapped) and (mapped[cursor, 0] != k2[j, 0] or mapped[cursor, 1] != k2[j, 1]):
            cursor += 1
        assert cursor < len(mapped)
        total += 1
        good += xa.hamming_distance(d1[cursor], d2[j]) <= 64
        cursor += 1
    assert total > 30 and good >= total * 7 // 10


def test_hamming_metric_axioms(xa):
    # test_features_binary.cpp:190-203: naive per-bit count, d(a,a)=0, symmetry, triangle
    d = random_descriptors(40, 7)
    bits = np.unpackbits(d.view(np.uint8), axis=1)
    for i in range(0, 40, 7):
        for j in range(0, 40, 5):
            dij = xa.hamming_distance(d[i], d[j])
            assert dij == int(np.sum(bits[i] != bits[j]))
            assert dij == xa.hamming_distance(d[j], d[i])
            assert xa.hamming_distance(d[i], d[i]) == 0
            for k in range(0, 40, 13):
                assert dij <= xa.hamming_distance(d[i], d[k]) + xa.hamming_distance(d[k], d[j])
    # the device matcher's distances are the same counts
    m = xa.match_hamming(d[:20], d[20:], 1.0)
    for r in m:
        assert int(r["distance"]) == xa.hamming_distance(d[int(r["idx_a"])], d[20 + int(r["idx_b"])])


def test_ratio_shrinkage_only_removes_matches(xa):
    # test_features_binary.cpp:248-265
    da, db = random_descriptors(200, 11), random_descriptors(200, 22)
    prev = None
    for ratio in (1.0, 0.9, 0.75, 0.5):
        cur = xa.match_hamming(da, db, ratio)
        pairs = {(int(r["idx_a"]), int(r["idx_b"])) for r in cur}
        if prev is not None:
            assert pairs <= prev
        prev = pairs


@pytest.mark.parametrize("t,phi,s", [(2.0, 0.3, 1.0), (4.0, 1.2, 1.5), (1.0, 0.0, 0.7)])
def test_simulation_determinant(xa, t, phi, s):
    # test_geometry.cpp:205-216: det = s^2 / t and x compressed by 1/t
    m = xa.simulation_from_params(xa.AffineParams(tilt=t, phi=phi, scale=s))
    assert np.linalg.det(m[:2, :2]) == pytest.approx(s * s / t, rel=1e-12)


def test_simulation_compresses_tilt_direction(xa):
    # test_geometry.cpp:205-216
    m = xa.simulation_from_params(xa.AffineParams(tilt=2.0))
    assert m[0, 0] == pytest.approx(0.5, rel=1e-12) and m[1, 1] == pytest.approx(1.0, rel=1e-12)
    ms = xa.simulation_from_params(xa.AffineParams(tilt=2.0, scale=3.0))
    assert ms[0, 0] * ms[1, 1] - ms[0, 1] * ms[1, 0] == pytest.approx(4.5, rel=1e-9)


def test_lanczos_round_trip(xa, port):
    # test_warp.cpp:127-151: warp, undo in the same convention, MAE < 2
    img = xa.gaussian_blur(port.make_texture(96, 96, 11), 1.0)
    m = xa.affine_from_params(xa.AffineParams(psi=0.3, tilt=1.6, phi=0.8, scale=1.2))
    w1 = xa.warp_lanczos(img, m, 4)
    shift = np.array([[1.0, 0.0, w1.tx], [0.0, 1.0, w1.ty], [0.0, 0.0, 1.0]])
    w2 = xa.warp_lanczos(w1.image, xa.invert(shift @ m), 4)
    ox, oy = int(round(w2.tx)), int(round(w2.ty))
    h, w = img.shape
    H, W = w2.image.shape
    err = []
    for y in range(12, h - 12):
        for x in range(12, w - 12):
            yy, xx = min(max(y + oy, 0), H - 1), min(max(x + ox, 0), W - 1)
            err.append(abs(float(w2.image[yy, xx]) - float(img[y, x])))
    assert float(np.mean(err)) < 2.0
