"""Edge shapes through the measured coarse path, pinned exactly like
test_gpu_pinned.py (the device's own uint8 views through the oracle's detect ->
filter_to_content -> describe -> match_hamming; counts EQUAL): image sides that
are not multiples of the 4-pixel / 16-byte staging units, reference and target
images of different sizes, images too small for any keypoint (every view's scan
region is empty: the reference returns zero counts and best index 0,
pipeline.cpp:142-150), and ragged batches of such pairs against their
single-pair runs."""
import math

import numpy as np
import pytest

from test_gpu_pinned import _check

pytestmark = pytest.mark.gpu


def _pair(w, h, seed, tilt=2.0, psi=25.0):
    from paper_2503_03479_b200 import synth
    return synth.pair(w, h, seed, (1.0, 0.0, 0.0), (tilt, 0.0, math.radians(psi)))


@pytest.mark.parametrize("mode", ["nearest", "lanczos"])
@pytest.mark.parametrize("size", [(331, 257), (517, 203), (254, 389)])
def test_odd_sizes_exact(xa, port, size, mode):
    a, b = _pair(size[0], size[1], seed=41)
    assert a.shape == (size[1], size[0])
    _check(xa, port, a, b, xa.build_param_grid(xa.GridConfig(n=3)), 400, 0.8, mode)


def test_unequal_reference_and_target_exact(xa, port):
    a, b = _pair(402, 301, seed=43)
    b = np.ascontiguousarray(b[7:236, 11:330])  # 319 x 229 target
    got = _check(xa, port, a, b, xa.build_param_grid(xa.GridConfig(n=3)), 400, 0.8, "lanczos")
    assert got.max() > 0


@pytest.mark.parametrize("mode", ["nearest", "lanczos"])
def test_images_too_small_for_keypoints(xa, port, mode):
    a, b = _pair(33, 29, seed=45)
    grid = xa.build_param_grid(xa.GridConfig(n=3))
    got = _check(xa, port, a, b, grid, 400, 0.8, mode)
    r = xa.coarse_search(a, b, grid, 400, 0.8, warp_mode=mode)
    assert r.best_index == 0 and r.best_count == 0


def test_full_grid_on_an_odd_size_exact(xa, port):
    # the 43-entry default grid (tilts up to 4 sqrt 2: the widest view frames,
    # separable and general Lanczos views, border tiles on every side)
    a, b = _pair(611, 377, seed=47, tilt=3.0, psi=70.0)
    _check(xa, port, a, b, xa.build_param_grid(xa.GridConfig()), 600, 0.8, "lanczos")


@pytest.mark.parametrize("mode", ["nearest", "lanczos"])
def test_ragged_batch_of_odd_pairs(xa, port, mode, monkeypatch):
    monkeypatch.setenv("XA_BATCH_PAIRS", "2")  # chunks of 2 + a remainder chunk
    pairs = [_pair(331, 257, seed=51 + i, tilt=1.5 + 0.5 * i) for i in range(5)]
    grid = xa.build_param_grid(xa.GridConfig(n=3))
    eng = xa.Engine(0)
    res = xa.coarse_search_batch([a for a, _ in pairs], [b for _, b in pairs], grid, 400, 0.8,
                                 warp_mode=mode, engine=eng)
    for (a, b), r in zip(pairs, res):
        one = xa.coarse_search(a, b, grid, 400, 0.8, warp_mode=mode, engine=eng)
        assert [c for _, c in r.per_entry_counts] == [c for _, c in one.per_entry_counts]
        assert r.per_entry_keypoints == one.per_entry_keypoints
        assert r.best_index == one.best_index
