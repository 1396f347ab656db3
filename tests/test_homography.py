"""Geometric verification (homography.hpp:27-39) through the C-ABI, host code.

The reference's homography.cpp needs Eigen (absent), so it cannot be compiled
as an oracle ("parity unpinned" for RANSAC: DESIGN.md §2); these are the
reference's own test cases (proj/tests/test_homography.cpp) with the same
generator: std::mt19937_64 + std::uniform_real_distribution as libstdc++ draws
them (generate_canonical<double, 53>: one 64-bit draw / 2^64). The order in
which the reference's project(h, u(rng), u(rng)) evaluates its arguments is
unspecified in C++, so the point sets may be x/y-swapped relative to the
reference build; the asserted properties do not depend on it."""
import numpy as np
import pytest

import paper_2503_03479_b200 as xa
from _mt64 import MT64


def uniform(rng, a, b):
    r = float(rng()) / 18446744073709551616.0
    if r >= 1.0:
        r = np.nextafter(1.0, 0.0)
    return r * (b - a) + a


def sample_homography():
    return np.array([[1.2, 0.1, 30.0], [-0.15, 0.9, -12.0], [4e-4, -2e-4, 1.0]])


def project(h, x, y):
    w = h[2, 0] * x + h[2, 1] * y + h[2, 2]
    return (x, y, (h[0, 0] * x + h[0, 1] * y + h[0, 2]) / w, (h[1, 0] * x + h[1, 1] * y + h[1, 2]) / w)


def exact_correspondences(h, n, seed):
    rng = MT64(seed)
    out = []
    for _ in range(n):
        x = uniform(rng, 10.0, 500.0)
        y = uniform(rng, 10.0, 500.0)
        out.append(project(h, x, y))
    return out


def check_equal_normalized(a, b, tol):
    assert a[2, 2] != 0 and b[2, 2] != 0
    assert np.abs(a / a[2, 2] - b / b[2, 2]).max() < tol


def test_dlt_four_exact_points():
    h = sample_homography()
    pts = [project(h, 10, 10), project(h, 400, 20), project(h, 30, 380), project(h, 420, 410)]
    check_equal_normalized(xa.fit_homography_dlt(pts), h, 1e-6)


def test_dlt_many_exact_points():
    h = sample_homography()
    check_equal_normalized(xa.fit_homography_dlt(exact_correspondences(h, 40, 5)), h, 1e-6)


def test_dlt_rejects_fewer_than_four():
    with pytest.raises(xa.HomographyError):
        xa.fit_homography_dlt([(0, 0, 0, 0), (1, 0, 1, 0), (0, 1, 0, 1)])


def test_ransac_noiseless_eight():
    h = sample_homography()
    r, inl = xa.estimate_homography_ransac(exact_correspondences(h, 8, 11))
    check_equal_normalized(r, h, 1e-6)
    assert len(inl) == 8


def test_ransac_rejects_gross_outliers():
    h = sample_homography()
    pts = exact_correspondences(h, 8, 13) + [(50, 60, 900, 900), (100, 200, -400, 777), (321, 45, 0, 0),
                                             (222, 333, 1234, -55)]
    r, inl = xa.estimate_homography_ransac(pts)
    check_equal_normalized(r, h, 1e-6)
    assert inl.tolist() == list(range(8))


def test_ransac_minimal_case():
    h = sample_homography()
    r, inl = xa.estimate_homography_ransac(exact_correspondences(h, 4, 17))
    check_equal_normalized(r, h, 1e-5)
    assert len(inl) == 4


def test_ransac_errors():
    h = sample_homography()
    with pytest.raises(xa.HomographyError):
        xa.estimate_homography_ransac(exact_correspondences(h, 3, 19))
    junk = [(float(i), 2.0 * i, float(7 * i), float(i)) for i in range(12)]
    with pytest.raises(xa.HomographyError, match="no consensus"):
        xa.estimate_homography_ransac(junk)


def test_ransac_seed_deterministic():
    h = sample_homography()
    pts = exact_correspondences(h, 30, 29)
    rng = MT64(31)
    for _ in range(10):
        # argument evaluation order of the brace initialiser: left to right
        a, b, c, d = (uniform(rng, -800.0, 800.0) for _ in range(4))
        pts.append((a + 900, b + 900, c, d))
    r1, i1 = xa.estimate_homography_ransac(pts, seed=123)
    r2, i2 = xa.estimate_homography_ransac(pts, seed=123)
    assert np.array_equal(r1, r2) and np.array_equal(i1, i2)
    check_equal_normalized(r1, h, 1e-5)


def test_ransac_moderate_noise():
    h = sample_homography()
    rng = MT64(37)
    pts = []
    for _ in range(60):
        x = uniform(rng, 10.0, 500.0)
        y = uniform(rng, 10.0, 500.0)
        p = list(project(h, x, y))
        p[2] += uniform(rng, -0.5, 0.5)
        p[3] += uniform(rng, -0.5, 0.5)
        pts.append(tuple(p))
    for _ in range(20):
        a, b, c, d = (uniform(rng, 10.0, 500.0) for _ in range(4))
        pts.append((a, b, c + 600, d + 600))
    _, inl = xa.estimate_homography_ransac(pts)
    assert len(inl) >= 55 and np.all(inl < 60)


def test_ransac_inlier_capacity_and_threshold():
    h = sample_homography()
    pts = exact_correspondences(h, 50, 3)
    _, inl = xa.estimate_homography_ransac(pts, threshold=1e-3, seed=7)
    assert len(inl) == 50
