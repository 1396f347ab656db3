"""GPU parity of view simulation (antialias_tilt, warp_nearest, warp_lanczos)
against the oracle, plus the reference's own warp tests restated
(proj/tests/test_warp.cpp). Tolerances (north_star): views within 0.5 on the
0-255 scale before rounding; uint8 views identical except where the oracle's
value sits within a rounding tie (|v - (k + 0.5)| < TIE)."""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

BLUR_TOL = 2e-3     # pipeline blur stencil (float accumulation) vs the reference's double sum
LANCZOS_TOL = 2e-2  # float Lanczos-4 vs the reference's double Lanczos (0-255 scale)
TIE = 0.05          # uint8 disagreements are allowed only this close to k + 0.5


def _tex(port, w, h, s):
    return port.make_texture(w, h, s)


@pytest.mark.parametrize("t,phi", [(1.0, 0.3), (math.sqrt(2), 0.0), (2.0, 0.6), (2.0, 0.0),
                                   (2 * math.sqrt(2), 1.3), (4.0, 2.5), (4 * math.sqrt(2), 0.9)])
def test_antialias_tilt(xa, port, t, phi):
    img = _tex(port, 97, 83, 5)
    got = xa.antialias_tilt(img, t, phi)
    want = port.antialias_tilt(img, t, phi)
    assert got.shape == want.shape
    # the reference-facing blur replays the reference's double arithmetic
    assert np.array_equal(got, want), np.max(np.abs(got - want))


@pytest.mark.parametrize("t,phi", [(2.0, 0.6), (4 * math.sqrt(2), 2.2)])
def test_antialias_tilt_large_coordinates(xa, port, t, phi):
    """Per-pixel tap coordinates x + i*dx lose low bits of i*dx at large x
    (warp.cpp:152); the device follows the reference there too."""
    img = _tex(port, 1500, 40, 8)
    assert np.array_equal(xa.antialias_tilt(img, t, phi), port.antialias_tilt(img, t, phi))


def test_antialias_impulse_rows_only(xa):
    # test_warp.cpp:208-230: phi=0 blurs rows only, 1-D Gaussian response
    img = np.zeros((33, 33), np.float32)
    img[16, 16] = 255.0
    out = xa.antialias_tilt(img, 2.0, 0.0)
    sigma = 0.8 * math.sqrt(3.0)
    r = math.ceil(3 * sigma)
    k = np.exp(-0.5 * np.arange(-r, r + 1) ** 2 / sigma ** 2)
    k /= k.sum()
    for x in range(33):
        d = x - 16
        want = 255.0 * k[d + r] if abs(d) <= r else 0.0
        assert out[16, x] == pytest.approx(want, rel=1e-4, abs=1e-4)
    mask = np.ones(33, bool)
    mask[16] = False
    assert np.all(out[mask] == 0.0)


def test_antialias_identity_and_errors(xa, port):
    img = _tex(port, 32, 32, 4)
    assert np.array_equal(xa.antialias_tilt(img, 1.0, 0.7), img)
    with pytest.raises(xa.GeometryError):
        xa.antialias_tilt(img, 0.5, 0.0)


def test_nearest_exact_on_grid(xa, port):
    # warp_nearest is a pure copy: identical frames and pixels for every grid view
    img = _tex(port, 150, 110, 6)
    for p in port.build_grid():
        m = port.simulation_from_params(p)
        got = xa.warp_nearest(img, m)
        want = port.warp(img, m, "nearest")
        assert np.array_equal(got.image, want[0])
        assert (got.tx, got.ty) == (want[1], want[2])
        assert np.array_equal(got.forward, want[3])


def test_nearest_kats(xa, port):
    img = _tex(port, 40, 30, 9)
    w = xa.warp_nearest(img, np.eye(3))
    assert w.tx == 0 and w.ty == 0 and np.array_equal(w.image, img)
    src = np.array([[10 * x + y for x in range(8)] for y in range(4)], np.float32)
    w = xa.warp_nearest(src, np.diag([2.0, 1.0, 1.0]))
    assert w.image.shape == (4, 16)
    for x in range(16):
        assert np.array_equal(w.image[:, x], src[:, int(math.floor((x + 0.5) / 2.0))])
    src = (1 + 3 * np.arange(4)[:, None] + np.arange(3)[None, :]).astype(np.float32)
    rot = np.array([[0.0, -1.0, 0.0], [1.0, 0.0, 0.0], [0.0, 0.0, 1.0]])
    rot[0, 0] = rot[1, 1] = math.cos(math.pi / 2)
    w = xa.warp_nearest(src, rot)
    assert w.image.shape == (3, 4)
    for v in range(3):
        for u in range(4):
            assert w.image[v, u] == src[3 - u, v]
    m = np.eye(3)
    m[0, 0] = m[0, 1] = 0.0
    with pytest.raises(xa.GeometryError):
        xa.warp_nearest(_tex(port, 32, 32, 7), m)


def test_lanczos_grid_tolerance(xa, port):
    img = port.antialias_tilt(_tex(port, 150, 110, 8), 2.0, 0.6)
    worst = 0.0
    for p in port.build_grid():
        m = port.simulation_from_params(p)
        got = xa.warp_lanczos(img, m)
        want = port.warp(img, m, "lanczos")
        assert np.array_equal(got.forward, want[3]) and got.image.shape == want[0].shape
        worst = max(worst, float(np.max(np.abs(got.image - want[0]))))
    assert worst <= LANCZOS_TOL


def test_lanczos_kats(xa, port):
    img = _tex(port, 48, 36, 5)
    w = xa.warp_lanczos(img, np.eye(3))
    assert np.allclose(w.image, img, rtol=1e-5, atol=1e-4)
    const = np.full((64, 64), 77.0, np.float32)
    p = xa.AffineParams(tilt=2.0, phi=0.6, scale=1.5)
    w = xa.warp_lanczos(const, xa.affine_from_params(p))
    back = xa.invert(w.forward)
    ys, xs = np.mgrid[0:w.image.shape[0], 0:w.image.shape[1]]
    sx = back[0, 0] * xs + back[0, 1] * ys + back[0, 2]
    sy = back[1, 0] * xs + back[1, 1] * ys + back[1, 2]
    inner = (sx >= 4) & (sx <= 59) & (sy >= 4) & (sy <= 59)
    assert inner.sum() > 500
    assert np.allclose(w.image[inner], 77.0, rtol=1e-5)
    t = np.array([[1, 0, 3], [0, 1, -2], [0, 0, 1]], np.float64)
    src = _tex(port, 40, 40, 6)
    a, b = xa.warp_nearest(src, t), xa.warp_lanczos(src, t)
    assert np.allclose(a.image, b.image, rtol=1e-5, atol=1e-4)


def test_coarse_views_uint8(xa, port):
    """Device pipeline views (blur -> resample -> uint8) against the oracle's
    float views quantised with lround: disagreements only at rounding ties."""
    import ctypes as C
    import torch
    src = np.clip(np.rint(_tex(port, 160, 120, 11)), 0, 255).astype(np.uint8)
    grid = port.build_grid()
    eng = xa.Engine(0)
    for mode, tol in (("nearest", BLUR_TOL), ("lanczos", LANCZOS_TOL)):
        m = 0 if mode == "nearest" else 1
        offs, ws, hs, total = eng.simulate_views_plan(160, 120, grid, m)
        d_src = torch.from_numpy(src).cuda()
        d_out = torch.zeros(total, dtype=torch.uint8, device="cuda")
        eng.simulate_views_device(d_src.data_ptr(), 160, 120, grid, m, d_out.data_ptr())
        torch.cuda.synchronize()
        out = d_out.cpu().numpy()
        for i, p in enumerate(grid):
            fl = port.antialias_tilt(src.astype(np.float32), p[1], p[2])
            want, *_ = port.warp(fl, port.simulation_from_params(p), mode)
            got = out[offs[i]:offs[i] + ws[i] * hs[i]].reshape(hs[i], ws[i])
            assert got.shape == want.shape
            q = np.clip(np.floor(want + 0.5), 0, 255).astype(np.uint8)
            bad = got != q
            assert np.all(np.abs(got.astype(float) - want)[bad] <= 0.5 + tol)
            frac = want[bad] - np.floor(want[bad])
            assert np.all(np.abs(frac - 0.5) < TIE), (mode, i, want[bad][:5], got[bad][:5])
    eng.close()


@pytest.mark.parametrize("hname", ["synth_mild", "synth_strong"])
def test_synth_warp_case_golden(xa, golden, hname):
    """synth_warp_case (eval.cpp:101-141) on the device against the fixtures the
    reference itself produced: composed homography exact, image within the
    Lanczos tolerance, uint8 output = lround + clamp except at rounding ties."""
    want = golden[hname]
    got, comp = xa.synth_warp_case(golden["synth_in"], golden[f"{hname}_h"])
    assert np.array_equal(comp, golden[f"{hname}_composed"])
    assert got.shape == want.shape and got.dtype == np.float32
    assert np.max(np.abs(got - want)) <= LANCZOS_TOL
    assert np.array_equal(got == 0, want == 0)  # same content domain
    u8, comp2 = xa.synth_warp_case(golden["synth_in"], golden[f"{hname}_h"], out="u8")
    assert np.array_equal(comp2, comp) and u8.dtype == np.uint8
    q = np.clip(np.floor(want.astype(np.float64) + 0.5), 0, 255).astype(np.uint8)
    bad = u8 != q
    frac = want[bad] - np.floor(want[bad])
    assert np.all(np.abs(frac - 0.5) < TIE)


def test_synth_warp_case_large(xa, port):
    img = _tex(port, 320, 240, 13)
    hm = np.array([[0.85, -0.3, 20.0], [0.25, 0.9, -10.0], [6e-4, -4e-4, 1.0]])
    got, comp = xa.synth_warp_case(img, hm)
    want, wcomp = port.synth_warp_case(img, hm)
    assert np.array_equal(comp, wcomp) and got.shape == want.shape
    assert np.max(np.abs(got - want)) <= LANCZOS_TOL


def test_synth_warp_case_errors(xa, port):
    img = _tex(port, 40, 30, 2)
    with pytest.raises(xa.EvalError, match="degenerate homography for synthetic warp"):
        xa.synth_warp_case(img, np.diag([1.0, 1.0, 0.0]))
    with pytest.raises(xa.EvalError, match="unbounded"):
        xa.synth_warp_case(img, np.array([[1, 0, 0], [0, 1, 0], [-0.02535, 0, 1.0]]))
