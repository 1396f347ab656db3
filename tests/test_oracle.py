"""Pins the C restatement (oracle/xa_oracle.c) before it is trusted as the checker.

1. Against tests/golden/golden.npz, generated from the reference library itself
   (tools/make_golden.py) — runs everywhere.
2. Against oracle/_ref/libxaref.so (the reference compiled from its own sources)
   on more seeds and sizes — runs where the reference was built.
Every comparison is exact (bit equality); there is no tolerance in the oracle.
"""
import math

import numpy as np
import pytest

from _mt64 import MT64, random_descriptors


def test_mt19937_64_known_answer():
    rng = MT64(5489)
    for _ in range(9999):
        rng()
    assert rng() == 9981545732273789042


def test_pattern_checksum_pinned(port, golden):
    # proj/tests/test_features_binary.cpp:56-58
    assert port.pattern_checksum() == 0xA47E0017C161E6D8
    assert np.array_equal(port.pattern(), golden["pattern"])


def test_texture_generator(port, golden):
    assert np.array_equal(port.make_texture(64, 48, 3), golden["texture_64x48_s3"])
    import hashlib
    for w, h, s in [(128, 128, 8), (200, 160, 9), (256, 256, 15), (31, 31, 7)]:
        d = hashlib.sha256(port.make_texture(w, h, s).tobytes()).digest()
        assert d == golden[f"texture_hash_{w}x{h}_s{s}"].tobytes()


def test_param_grid(port, golden):
    g = port.build_grid()
    assert len(g) == 43  # test_geometry.cpp:158-182
    assert np.array_equal(g, golden["grid_default"])
    assert np.array_equal(port.build_grid(n=3), golden["grid_n3"])
    assert len(golden["grid_n3"]) == 18
    assert np.array_equal(port.build_grid(delta_s=0.0), golden["grid_ds0"])
    counts = [int(np.sum(np.isclose(g[:, 1], math.sqrt(2) ** k))) for k in range(6)]
    assert counts == [1, 4, 5, 8, 10, 15]


def test_antialias(port, golden):
    img = golden["aa_in"]
    assert np.array_equal(port.antialias_tilt(img, 2.0, 0.0), golden["aa_t2_phi0"])
    assert np.array_equal(port.antialias_tilt(img, 2.0, 0.6), golden["aa_t2_phi06"])
    assert np.array_equal(port.antialias_tilt(img, 4 * math.sqrt(2), 1.1), golden["aa_t4s2_phi1"])
    assert np.array_equal(port.antialias_tilt(img, 1.0, 0.7), img)


@pytest.mark.parametrize("mname", ["rot90", "stretch2", "sim_t2_phi36_s2", "sim_t28_phi1_s15"])
@pytest.mark.parametrize("mode", ["nearest", "lanczos"])
def test_warps(port, golden, mname, mode):
    im, tx, ty, fwd = port.warp(golden["warp_in"], golden[f"mat_{mname}"], mode)
    assert np.array_equal(im, golden[f"warp_{mode}_{mname}"])
    assert np.array_equal(np.array([tx, ty, *fwd.reshape(-1)]), golden[f"warp_{mode}_{mname}_frame"])


@pytest.mark.parametrize("hname", ["synth_mild", "synth_strong"])
def test_synth_warp_case(port, golden, hname):
    """eval.cpp:101-141 restated: image and composed homography bit-identical."""
    im, comp = port.synth_warp_case(golden["synth_in"], golden[f"{hname}_h"])
    assert np.array_equal(im, golden[hname])
    assert np.array_equal(comp, golden[f"{hname}_composed"])


def test_synth_warp_case_errors(port):
    """The reference's EvalError cases (eval.cpp:110, :118-119, :129-134)."""
    from oracle.oracle import OracleError
    img = port.make_texture(40, 30, 2)
    with pytest.raises(OracleError, match="degenerate homography for synthetic warp"):
        port.synth_warp_case(img, np.diag([1.0, 1.0, 0.0]))
    # w -> 0 between the corners: the image of the frame is unbounded
    with pytest.raises(OracleError, match="unbounded"):
        port.synth_warp_case(img, np.array([[1, 0, 0], [0, 1, 0], [-0.02535, 0, 1.0]]))


def test_port_equals_reference_synth_warp(port, ref):
    img = port.make_texture(120, 90, 21)
    for hm in ([[1.1, 0.2, -5.0], [-0.15, 0.95, 7.0], [1e-3, 5e-4, 1.0]],
               [[0.5, 0.0, 0.0], [0.0, 0.5, 0.0], [0.0, 0.0, 1.0]], np.eye(3)):
        a, ca = port.synth_warp_case(img, hm)
        b, cb = ref.synth_warp_case(img, hm)
        assert np.array_equal(a, b) and np.array_equal(ca, cb)


def test_orb_detect_describe(port, golden):
    tex = port.make_texture(128, 128, 8)
    kps = port.detect(tex, 200)
    assert np.array_equal(kps, golden["orb_tex128_kps"])
    k2, d2 = port.describe(tex, kps)
    assert np.array_equal(k2, golden["orb_tex128_desc_kps"])
    assert np.array_equal(d2, golden["orb_tex128_desc"])
    cb = port.make_checkerboard(256, 256, 32)
    kc = port.detect(cb, 1000)
    assert np.array_equal(kc, golden["orb_checker_kps"])
    assert np.array_equal(port.describe(cb, kc)[1], golden["orb_checker_desc"])
    t256 = port.make_texture(256, 256, 15)
    assert np.array_equal(port.detect(t256, 1000), golden["orb_tex256_kps_all"])
    assert np.array_equal(port.detect(t256, 50), golden["orb_tex256_kps_cap50"])


def test_orb_auto_relax(port, golden):
    relax = port.make_texture(200, 200, 21) * np.float32(0.12) + np.float32(90)
    k = port.detect(relax, 1000)
    assert np.array_equal(k, golden["orb_relax_kps"])


def test_orb_edge_cases(port):
    assert len(port.detect(np.full((128, 128), 100, np.float32), 1000)) == 0
    assert len(port.detect(port.make_texture(31, 31, 7), 1000)) == 0
    assert len(port.detect(port.make_texture(64, 64, 7), 0)) == 0


@pytest.mark.parametrize("r", [0.6, 0.75, 0.9, 1.0])
def test_matcher_kat(port, golden, r):
    da, db = golden["desc_s101"], golden["desc_s202"]
    assert np.array_equal(da, random_descriptors(500, 101))
    assert np.array_equal(port.match(da, db, r), golden[f"match_s101_s202_r{r}"])


def test_matcher_acceptance_kat(port, golden):
    a, b = golden["desc_s161_a"], golden["desc_s161_b"]
    assert np.array_equal(port.match(a, b, 0.75), golden["match_s161_r0.75"])
    assert np.array_equal(port.match(a, b, 0.6), golden["match_s161_r0.6"])


def test_coarse_search(port, golden):
    for mode in ("nearest", "lanczos"):
        c, kpc, best = port.coarse_search(golden["coarse_in"], golden["coarse_tgt"],
                                          golden["coarse_grid"], 300, 0.75, mode, threads=2)
        assert np.array_equal(c, golden[f"coarse_{mode}_counts"])
        assert best == int(golden[f"coarse_{mode}_best"][0])


# ---------------------------------------------------------------- vs reference

def _canon_kps(k):
    """The reference sorts with std::sort (unstable) on (response, y, x):
    keypoints that differ only in orientation have no defined order."""
    k = np.asarray(k)
    return k[np.lexsort((k[:, 3], k[:, 0], k[:, 1], -k[:, 2]))]


@pytest.mark.parametrize("seed,w,h", [(1, 160, 128), (2, 256, 200), (3, 97, 131)])
def test_port_equals_reference_sift(port, ref, seed, w, h):
    """detect_dog_keypoints / describe_gradient (sift.cpp:290-386): the C
    restatement equals the reference bit for bit (keypoints as a multiset)."""
    img = ref.make_texture(w, h, seed)
    kr, kp = ref.detect_dog(img, 500), port.detect_dog(img, 500)
    assert len(kr) > 30 and np.array_equal(_canon_kps(kr), _canon_kps(kp))
    dr, dp = ref.describe_gradient(img, kr), port.describe_gradient(img, kr)
    assert len(dr[0]) > 20
    assert np.array_equal(dr[0], dp[0]) and np.array_equal(dr[1], dp[1])
    assert len(port.detect_dog(img[:60, :60], 100)) == 0  # < 64 px (sift.hpp:12)


def test_port_equals_reference_match_ratio(port, ref):
    """match_ratio (sift.cpp:388-418): the C restatement equals the reference
    bit for bit, including exact duplicates, ties and the missing-second rule."""
    rng = np.random.default_rng(7)
    a = (rng.random((120, 128)) * 40).astype(np.float32)
    b = (rng.random((150, 128)) * 40).astype(np.float32)
    b[::5] = a[:30] + rng.normal(0, 1.0, (30, 128)).astype(np.float32)
    b[7] = b[8]
    b[11] = a[3]
    for r in (0.6, 0.8, 1.0):
        x, y = port.match_ratio(a, b, r), ref.match_ratio(a, b, r)
        assert np.array_equal(x, y)
    assert np.array_equal(port.match_ratio(a[:3], b[:1], 0.75), ref.match_ratio(a[:3], b[:1], 0.75))
    assert len(port.match_ratio(a[:0], b, 0.75)) == 0


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_port_equals_reference_orb(port, ref, seed):
    rng = np.random.default_rng(seed)
    w, h = int(rng.integers(60, 300)), int(rng.integers(60, 300))
    img = ref.make_texture(w, h, seed)
    for mp in (50, 300, 1000):
        kr = ref.detect(img, mp)
        kp = port.detect(img, mp)
        assert np.array_equal(kr, kp)
        dr = ref.describe(img, kr)
        dp = port.describe(img, kp)
        assert np.array_equal(dr[0], dp[0]) and np.array_equal(dr[1], dp[1])


def test_port_equals_reference_views(port, ref):
    img = ref.make_texture(150, 110, 4)
    for p in ref.build_grid():
        a = ref.antialias_tilt(img, p[1], p[2])
        assert np.array_equal(a, port.antialias_tilt(img, p[1], p[2]))
        m = ref.simulation_from_params(p)
        assert np.array_equal(m, port.simulation_from_params(p))
        for mode in ("nearest", "lanczos"):
            x, y = ref.warp(a, m, mode), port.warp(a, m, mode)
            assert np.array_equal(x[0], y[0]) and x[1:3] == y[1:3]


def test_port_equals_reference_coarse(port, ref):
    img = ref.make_texture(160, 160, 7)
    g = ref.build_grid()
    for mode in ("nearest", "lanczos"):
        a = ref.coarse_search(img, img, g, 500, 0.75, mode, threads=8)
        b = port.coarse_search(img, img, g, 500, 0.75, mode, threads=8)
        assert np.array_equal(a[0], b[0]) and a[2] == b[2]
