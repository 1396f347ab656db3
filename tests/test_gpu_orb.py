"""GPU ORB (detect_oriented_corners, describe_binary) bit-exact against the
oracle and the reference-generated golden fixtures, plus the reference's own
binary-feature tests restated (proj/tests/test_features_binary.cpp)."""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def kp_arr(k):
    return np.asarray(k).view(np.float32).reshape(-1, 5)


def assert_same_kps(got, want):
    g, w = kp_arr(got), np.asarray(want, np.float32).reshape(-1, 5)
    assert g.shape == w.shape, (g.shape, w.shape)
    if not np.array_equal(g, w):
        bad = np.where(np.any(g != w, axis=1))[0]
        raise AssertionError(f"{len(bad)} keypoints differ; first {bad[:5]}: {g[bad[:3]]} vs {w[bad[:3]]}")


def test_golden_detect_describe(xa, golden):
    from oracle.oracle import Oracle  # noqa: F401  (golden comes from the reference)
    tex = golden["orb_tex128_kps"]
    port_img = None
    import oracle.oracle as O
    port_img = O.Oracle("port").make_texture(128, 128, 8)
    k = xa.detect_oriented_corners(port_img, 200)
    assert_same_kps(k, golden["orb_tex128_kps"])
    k2, d2 = xa.describe_binary(port_img, k)
    assert_same_kps(k2, golden["orb_tex128_desc_kps"])
    assert np.array_equal(d2, golden["orb_tex128_desc"])
    del tex


def test_golden_checker_and_cap(xa, port, golden):
    cb = port.make_checkerboard(256, 256, 32)
    k = xa.detect_oriented_corners(cb, 1000)
    assert_same_kps(k, golden["orb_checker_kps"])
    assert np.array_equal(xa.describe_binary(cb, k)[1], golden["orb_checker_desc"])
    assert len(k) >= 100  # test_features_binary.cpp:68-79
    t256 = port.make_texture(256, 256, 15)
    assert_same_kps(xa.detect_oriented_corners(t256, 1000), golden["orb_tex256_kps_all"])
    assert_same_kps(xa.detect_oriented_corners(t256, 50), golden["orb_tex256_kps_cap50"])


def test_golden_auto_relax(xa, port, golden):
    relax = port.make_texture(200, 200, 21) * np.float32(0.12) + np.float32(90)
    assert_same_kps(xa.detect_oriented_corners(relax, 1000), golden["orb_relax_kps"])


@pytest.mark.parametrize("seed", range(6))
def test_detect_describe_random_textures(xa, port, seed):
    rng = np.random.default_rng(100 + seed)
    w, h = int(rng.integers(64, 400)), int(rng.integers(64, 400))
    img = port.make_texture(w, h, seed + 30)
    if seed % 2:
        img = np.clip(np.rint(img), 0, 255)  # integer-valued (uint8 view) images too
    for mp in (100, 500, 2000):
        want = port.detect(img, mp)
        got = xa.detect_oriented_corners(img, mp)
        assert_same_kps(got, want)
        wk, wd = port.describe(img, want)
        gk, gd = xa.describe_binary(img, got)
        assert_same_kps(gk, wk)
        assert np.array_equal(gd, wd)


def test_synthetic_views_bit_exact(xa, port):
    """ORB on uint8 views from the BASELINE texture generator (the pipeline's inputs)."""
    from paper_2503_03479_b200 import synth
    a, b = synth.config1(seed=7)
    for img in (a, b):
        f = img.astype(np.float32)
        want = port.detect(f, 500)
        got = xa.detect_oriented_corners(f, 500)
        assert_same_kps(got, want)
        assert np.array_equal(xa.describe_binary(f, got)[1], port.describe(f, want)[1])


def test_edge_cases(xa, port):
    assert len(xa.detect_oriented_corners(np.full((128, 128), 100, np.float32), 1000)) == 0
    assert len(xa.detect_oriented_corners(port.make_texture(31, 31, 7), 1000)) == 0
    assert len(xa.detect_oriented_corners(port.make_texture(64, 64, 7), 0)) == 0
    k, d = xa.describe_binary(port.make_texture(64, 64, 7), np.zeros((0, 5), np.float32))
    assert len(k) == 0 and d.shape == (0, 4)


def test_describe_border_and_gain(xa, port):
    # test_features_binary.cpp:121-152
    img = port.make_texture(128, 128, 8)
    kps = kp_arr(xa.detect_oriented_corners(img, 200)).copy()
    kps = np.vstack([kps, [[5, 5, 0, 0, 1]]]).astype(np.float32)
    k1, d1 = xa.describe_binary(img, kps)
    k2, d2 = xa.describe_binary(img, kps)
    assert len(k1) < len(kps) and len(k1) > 0 and np.array_equal(d1, d2)
    assert np.all(kp_arr(k1)[:, 0] >= 20) and np.all(kp_arr(k1)[:, 1] >= 20)
    pk, pd = port.describe(img, kps)
    assert np.array_equal(d1, pd)
    img2 = port.make_texture(128, 128, 12)
    kk = xa.detect_oriented_corners(img2, 100)
    _, da = xa.describe_binary(img2, kk)
    _, db = xa.describe_binary(img2 * np.float32(0.5), kk)
    assert np.array_equal(da, db)


def test_describe_rotated_orientations(xa, port):
    # angles beyond [-pi, pi] exercise the glibc cosf/sinf fixup path
    img = port.make_checkerboard(256, 256, 32)
    k = kp_arr(xa.detect_oriented_corners(img, 300)).copy()
    for add in (0.0, math.pi / 6, 2.5, -4.0):
        kk = k.copy()
        kk[:, 3] = (kk[:, 3] + np.float32(add)).astype(np.float32)
        assert np.array_equal(xa.describe_binary(img, kk)[1], port.describe(img, kk)[1])


def test_trig_fixup_angles(xa, port):
    """Keypoint angles taken from the fixup table itself: the device must
    reproduce glibc's cosf/sinf-steered pattern exactly at those angles."""
    import re
    import pathlib
    inc = (pathlib.Path(xa.__file__).parent / "csrc" / "trig_fixups.inc").read_text()
    xs = [int(m, 16) for m in re.findall(r"\{0x([0-9a-f]{8})u", inc)][::7]
    ang = np.array(xs, np.uint32).view(np.float32)
    img = port.make_texture(160, 160, 3)
    kps = np.zeros((len(ang), 5), np.float32)
    kps[:, 0] = 80
    kps[:, 1] = 80
    kps[:, 3] = ang
    kps[:, 4] = 1
    assert np.array_equal(xa.describe_binary(img, kps)[1], port.describe(img, kps)[1])
