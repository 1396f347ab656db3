"""Reference selection (pipeline.cpp:70-120) and the ASIFT
baseline restatement (§8f row 2) on the CPU:
the host scaling coefficient of the product API and of the C restatement
against the reference's own known-answer cases (proj/tests/test_pipeline.cpp:
38-140, acceptance_main.cpp:396-411) and against the reference library itself."""
import math

import numpy as np
import pytest

from paper_2503_03479_b200 import api

MDT = [("idx_a", np.int32), ("idx_b", np.int32), ("distance", np.float32)]


def _kps(pts):
    k = np.zeros((len(pts), 5), np.float32)
    k[:, :2] = np.asarray(pts, np.float32)
    k[:, 4] = 1.0
    return k


def _matches(triples):
    m = np.zeros(len(triples), MDT)
    for i, (a, b, d) in enumerate(triples):
        m[i] = (a, b, d)
    return m


def _both(port, ka, kb, m):
    f, seg = api.scaling_coefficient(ka, kb, m)
    assert (f, seg) == port.scaling_coefficient(ka, kb, m)
    return f, seg


def test_self_matches_zero(port):
    k = _kps([(10 * i, 3 * i) for i in range(5)])
    f, _ = _both(port, k, k, _matches([(i, i, 50 + i) for i in range(5)]))
    assert f == 0.0


def test_half_shrink_positive(port):
    pts = [(0, 0), (40, 8), (10, 50), (60, 60), (25, 30), (5, 70), (70, 20), (45, 45)]
    a = _kps(pts)
    b = _kps([(x * 0.5, y * 0.5) for x, y in pts])
    f, _ = _both(port, a, b, _matches([(i, i, 100 + 10 * i) for i in range(8)]))
    assert f > 0.0


def test_six_match_hand_oracle(port):
    a = _kps([(0, 0), (3, 4), (10, 0), (0, 10), (6, 8), (20, 20)])
    b = _kps([(0, 0), (1.5, 2), (5, 0), (0, 5), (3, 4), (10, 10)])
    dist = [100, 200, 300, 400, 150, 250]
    f, seg = _both(port, a, b, _matches([(i, i, dist[i]) for i in range(6)]))
    expect = (10.0 - 5.0) * 0.75 + (math.sqrt(200.0) - math.sqrt(50.0)) * 0.3
    assert seg == 2 and abs(f - expect) < 1e-9


def test_negative_weight_clamped(port):
    a = _kps([(0, 0), (100, 0)])
    b = _kps([(0, 0), (10, 0)])
    f, _ = _both(port, a, b, _matches([(0, 0, 600), (1, 1, 700)]))
    assert f == 0.0


def test_needs_two_matches(port):
    k = _kps([(0, 0)])
    for m in (_matches([(0, 0, 10)]), _matches([])):
        with pytest.raises(api.PipelineError):
            api.scaling_coefficient(k, k, m)
        with pytest.raises(Exception):
            port.scaling_coefficient(k, k, m)
    with pytest.raises(api.PipelineError):
        api.scaling_coefficient(k, k, _matches([(0, 0, 1), (0, 3, 2)]))


def test_random_sets_equal_reference(port, ref):
    """Ties on distance (ordered by idx_a), float-precision segment lengths:
    the API's host arithmetic equals the reference library bit for bit."""
    rng = np.random.default_rng(5)
    for trial in range(20):
        na, nb, n = rng.integers(2, 60, size=3)
        ka = (rng.random((na, 5)) * 500).astype(np.float32)
        kb = (rng.random((nb, 5)) * 300).astype(np.float32)
        ia = rng.permutation(na)[: min(n, na)]
        m = np.zeros(len(ia), MDT)
        m["idx_a"], m["idx_b"] = ia, rng.integers(0, nb, len(ia))
        m["distance"] = np.round(rng.random(len(ia)) * 600, 0 if trial % 2 else 3)
        if len(m) < 2:
            continue
        want = ref.scaling_coefficient(ka, kb, m)
        assert api.scaling_coefficient(ka, kb, m) == want
        assert port.scaling_coefficient(ka, kb, m) == want


def test_select_reference_port_equals_reference(port, ref):
    """select_reference cases of test_pipeline.cpp:116-140, restatement vs library."""
    img = ref.make_texture(256, 256, 3)
    small = ref.resize_bilinear(img, 128, 128)
    d = ref.select_reference(img, small, 500)
    assert d == port.select_reference(img, small, 500)
    assert d[0] == 1 and d[1] > d[2] and d[3] > 0
    s = ref.select_reference(small, img, 500)
    assert s == port.select_reference(small, img, 500) and s[0] == 2
    same = ref.make_texture(160, 160, 5)
    t = port.select_reference(same, same, 400)
    assert t == ref.select_reference(same, same, 400) and t[0] == 1 and t[1] == t[2]
    big, sm = np.full((200, 200), 100, np.float32), np.full((100, 100), 100, np.float32)
    assert port.select_reference(big, sm)[0] == 1 == ref.select_reference(big, sm)[0]
    assert port.select_reference(sm, big)[0] == 2 == ref.select_reference(sm, big)[0]


def _rows(a):
    return a[np.lexsort(a.T[::-1])]


def test_asift_port_equals_reference(port, ref):
    """asift_baseline up to RANSAC (pipeline.cpp:242-343): the C restatement
    equals the reference library as a multiset of correspondences (keypoints
    of one extremum that differ only in orientation have no defined order in
    the reference, so two such matches can trade places)."""
    img = ref.make_texture(160, 128, 3)
    tgt = ref.warp(img, ref.affine_from_params([0.3, 1.3, 0.5, 1.0, 0, 0]), "lanczos")[0]
    g = ref.build_grid(n=2)
    a = ref.asift_correspondences(img, tgt, g, 300, 0.75)
    b = port.asift_correspondences(img, tgt, g, 300, 0.75)
    assert len(a) > 100 and np.array_equal(_rows(a), _rows(b))
    # a one-entry (identity) grid degenerates to plain fine matching
    # (test_pipeline.cpp:296-310)
    one = port.asift_correspondences(img, tgt, g[:1], 300, 0.75)
    k1, d1 = port.describe_gradient(img, port.detect_dog(img, 300))
    k2, d2 = port.describe_gradient(tgt, port.detect_dog(tgt, 300))
    assert len(one) == len(port.match_ratio(d1, d2, 0.75))
