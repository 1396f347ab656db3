"""Inputs the reference accepts that exceed the device's fast-path buffers.

detect_oriented_corners (orb.cpp:182-210) has no keypoint cap and its sort has
no tie limit, so the device path must give the reference's answer for
max_points above the shared-memory sort (kSortCap entries) and for images
where more than kSortCap keys tie at the N-th response; both go through the
global-memory selection k_select_big. Results are compared EXACTLY with the
oracle (keypoints: x, y, response, orientation, octave scale)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _same_keypoints(xa, port, img, n):
    got = np.asarray(xa.detect_oriented_corners(img, n)).view(np.float32).reshape(-1, 5)
    want = port.detect(img, n)
    assert got.shape == want.shape, (got.shape, want.shape)
    assert np.array_equal(got, want)
    return got


def test_max_points_above_sort_buffer(xa, port):
    from paper_2503_03479_b200 import synth
    a, _ = synth.config2(seed=7)
    k = _same_keypoints(xa, port, a.astype(np.float32), 12000)
    assert len(k) > 8192  # really beyond the shared-memory sort


def test_more_ties_than_sort_buffer(xa, port):
    # a 16x16 random block tiled to 2048x2048: every corner of the block
    # repeats 16384 times at level 0 with the identical response, so the
    # N-th response is tied far beyond kSortCap
    rng = np.random.default_rng(5)
    blk = rng.integers(0, 256, (16, 16)).astype(np.float32)
    img = np.ascontiguousarray(np.tile(blk, (128, 128)))
    k = _same_keypoints(xa, port, img, 1000)
    assert len(k) == 1000
    assert np.all(k[:, 2] == k[0, 2])  # the whole kept set is one tie group


def test_describe_many_keypoints(xa, port):
    from paper_2503_03479_b200 import synth
    a, _ = synth.config2(seed=8)
    f = a.astype(np.float32)
    k = port.detect(f, 10000)
    kk, d = xa.describe_binary(f, k)
    wk, wd = port.describe(f, k)
    assert np.array_equal(np.asarray(kk).view(np.float32).reshape(-1, 5), wk)
    assert np.array_equal(d, wd)


def test_coarse_large_max_points_exact(xa, port):
    """The reference coarse stage (float views, nearest) with max_points above
    the shared-memory sort: counts equal the oracle's coarse_search."""
    from paper_2503_03479_b200 import synth
    a, b = synth.config1(seed=4)
    f, bf = a.astype(np.float32), b.astype(np.float32)
    grid = port.build_grid(n=2)
    r = xa.coarse_search(f, bf, grid, 9000, 0.8, warp_mode="nearest")
    want, _, wbest = port.coarse_search(f, bf, grid, 9000, 0.8, "nearest", threads=16)
    got = np.array([c for _, c in r.per_entry_counts])
    assert np.array_equal(got, want) and r.best_index == wbest, (got, want)
