"""Reference selection and the fine-stage correspondences (pipeline.cpp:103-120,
154-190; SURVEY.md §8f rows 1+3) through the device SIFT + L2 matcher, against
the reference library and the C restatement.

The host arithmetic (scaling coefficient, content filter, back-mapping) is
bit-exact (tests/test_reference_selection.py); the device descriptors sit
within DESC_TOL of the reference's (test_gpu_sift.py), so a handful of ratio
decisions can flip. Asserted here: identical decisions, scaling coefficients
within F_TOL relative, correspondences agreeing on at least AGREE (positions within POS_TOL px)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

F_TOL = 0.05
AGREE = 0.97
POS_TOL = 1e-3


def test_select_reference_cases(xa, ref):
    # test_pipeline.cpp:116-140
    img = ref.make_texture(256, 256, 3)
    small = ref.resize_bilinear(img, 128, 128)
    for a, b, want in ((img, small, 1), (small, img, 2)):
        d = xa.select_reference(a, b, 500)
        r = ref.select_reference(a, b, 500)
        assert d.reference == r[0] == want
        assert d.f_forward == pytest.approx(r[1], rel=F_TOL)
        assert d.f_backward == pytest.approx(r[2], rel=F_TOL, abs=1.0)
        assert abs(d.segment_count - r[3]) <= max(2, r[3] // 20)
    same = ref.make_texture(160, 160, 5)
    d = xa.select_reference(same, same, 400)
    assert d.reference == 1 and d.f_forward == d.f_backward
    big, sm = np.full((200, 200), 100, np.float32), np.full((100, 100), 100, np.float32)
    assert xa.select_reference(big, sm).reference == 1
    assert xa.select_reference(sm, big).reference == 2


def test_scaling_on_device_features_equals_reference(xa, ref):
    """Same inputs (the device's own features and matches) -> the reference's
    scaling_coefficient and the API's agree bit for bit."""
    img = ref.make_texture(300, 240, 8)
    small = ref.resize_bilinear(img, 200, 160)
    k1, d1 = xa.fine_features(img, 600)
    k2, d2 = xa.fine_features(small, 600)
    m = xa.match_ratio(d1, d2, 0.75)
    assert len(m) > 20
    assert xa.scaling_coefficient(k1, k2, m) == ref.scaling_coefficient(k1, k2, m)


@pytest.mark.parametrize("p,size", [([0.3, 1.414, -0.9, 0.8, 0, 0], 256), ([0.0, 1.414, 0.5, 1.0, 0, 0], 320)])
def test_fine_correspondences_vs_restatement(xa, port, p, size):
    """fine_match up to RANSAC (pipeline.cpp:154-183) composed from the C
    restatement's stages vs the device path."""
    img = port.make_texture(size, size - 32, 12 if size == 256 else 4)
    tgt = port.warp(img, port.affine_from_params(p), "lanczos")[0]
    params = xa.AffineParams(psi=0.0, tilt=p[1], phi=p[2], scale=p[3])
    got, fwd = xa.fine_correspondences(img, tgt, params, max_points=800)

    pr = [0.0, p[1], p[2], p[3], 0.0, 0.0]
    filt = port.antialias_tilt(img, p[1], p[2])
    wimg, _, _, pfwd = port.warp(filt, port.simulation_from_params(pr), "lanczos", 4)
    assert np.array_equal(fwd, pfwd)
    back = port.invert(pfwd)
    kps = port.filter_to_content(port.detect_dog(wimg, 800), back, img.shape[1], img.shape[0], 4.0)
    wk, wd = port.describe_gradient(wimg, kps)
    tk, td = port.describe_gradient(tgt, port.detect_dog(tgt, 800))
    m = port.match_ratio(wd, td, 0.75)
    want = []
    for r in m:
        x, y = xa.map_point(back, float(wk[r["idx_a"], 0]), float(wk[r["idx_a"], 1]))
        want.append((x, y, float(tk[r["idx_b"], 0]), float(tk[r["idx_b"], 1])))
    want = np.asarray(want)
    assert len(want) > 20
    # the float Lanczos view sits within ~1e-4 of the reference's (different
    # summation order), which moves refined DoG positions by ~1e-4 px
    close = sum(np.abs(got[:, :4] - w).max(1).min() <= POS_TOL for w in want)
    worst = max(len(got), len(want))
    assert worst - close <= max(2, (1 - AGREE) * worst)


def _match_rows(got, want, tol):
    """How many rows of `want` have a row of `got` within tol (all 5 columns)."""
    if len(got) == 0:
        return 0
    return sum(np.abs(got - w).max(1).min() <= tol for w in want)


def test_asift_vs_restatement(xa, port):
    """asift_baseline up to RANSAC (pipeline.cpp:242-343): device views + SIFT
    + per-pair L2 matching + host duplicate merge, against the C restatement.
    Float views differ by ~1e-4 (summation order), so positions are compared
    within POS_TOL and descriptor distances within 0.05."""
    img = port.make_texture(160, 128, 3)
    tgt = port.warp(img, port.affine_from_params([0.3, 1.3, 0.5, 1.0, 0, 0]), "lanczos")[0]
    grid = xa.build_param_grid(xa.GridConfig(n=2))
    g = np.array([[p.psi, p.tilt, p.phi, p.scale, p.tx, p.ty] for p in grid.entries])
    want = port.asift_correspondences(img, tgt, g, 300, 0.75)
    got = xa.asift_correspondences(img, tgt, grid, 300, 0.75)
    assert len(want) > 100
    close = _match_rows(got[:, :4], want[:, :4], POS_TOL)
    worst = max(len(got), len(want))
    assert worst - close <= max(2, (1 - AGREE) * worst)
    # distances of position-matched rows agree to the float rounding of slightly
    # different descriptors (two rows can share a position: keypoints of one
    # extremum that differ only in orientation)
    for w in want:
        near = np.abs(got[:, :4] - w[:4]).max(1) <= POS_TOL
        if near.any():
            assert np.abs(got[near, 4] - w[4]).min() < 0.05


def test_asift_identity_grid_is_fine_matching(xa, port):
    # test_pipeline.cpp:296-310: a one-entry grid reduces to plain fine matching
    img = port.make_texture(200, 160, 4)
    tgt = port.warp(img, port.affine_from_params([0.2, 1.0, 0.0, 1.0, 0, 0]), "lanczos")[0]
    one = xa.ParamGrid([xa.AffineParams()], xa.GridConfig())
    got = xa.asift_correspondences(img, tgt, one, 400, 0.75)
    k1, d1 = xa.fine_features(img, 400)
    k2, d2 = xa.fine_features(tgt, 400)
    m = xa.match_ratio(d1, d2, 0.75)
    # the identity view is the source up to float rounding of the Lanczos sum
    # (about 1 ulp), which moves refined DoG positions by ~1e-5 px
    assert abs(len(got) - len(m)) <= 2 and len(m) > 20
    want = np.stack([k1[m["idx_a"], 0], k1[m["idx_a"], 1], k2[m["idx_b"], 0], k2[m["idx_b"], 1]], 1)
    assert _match_rows(got[:, :4], want, POS_TOL) >= len(want) - 2
