"""CPU checks of the C-ABI library: it builds for sm_100a, loads without a GPU,
exports every symbol include/xaffine_b200.h declares, and its host-side
geometry (which must match the reference bit-for-bit) equals the oracle."""
import ctypes as C
import math
import pathlib
import re

import numpy as np
import pytest

ROOT = pathlib.Path(__file__).resolve().parents[1]


@pytest.fixture(scope="module")
def lib():
    from paper_2503_03479_b200 import _lib, build
    build.build()
    return _lib.lib()


def declared_symbols():
    hdr = (ROOT / "include" / "xaffine_b200.h").read_text()
    return sorted(set(re.findall(r"^\s*(?:[\w\s\*]+?)\b(xa_\w+)\s*\(", hdr, re.M)))


def test_header_symbols_exported(lib):
    from paper_2503_03479_b200 import _lib
    names = declared_symbols()
    assert len(names) >= 25
    for n in names:
        assert hasattr(lib, n), n
        assert n in _lib.EXPORTS, f"{n} declared but not bound in _lib.py"


def test_sm100a_cubin_present():
    import subprocess
    so = ROOT / "paper_2503_03479_b200" / "libxa_b200.so"
    out = subprocess.run(["cuobjdump", "--list-elf", str(so)], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_pattern_and_trig_tables(lib):
    assert lib.xa_pattern_checksum() == 0xA47E0017C161E6D8
    assert lib.xa_trig_fixups() > 0


def test_param_grid_matches_oracle(lib, port):
    from paper_2503_03479_b200 import api
    for cfg in (api.GridConfig(), api.GridConfig(n=3), api.GridConfig(delta_s=0.0),
                api.GridConfig(a=1.7, n=4, b_deg=60.0, delta_s=0.25)):
        g = api.build_param_grid(cfg)
        arr = np.array([p.as_tuple() for p in g.entries])
        assert np.array_equal(arr, port.build_grid(cfg.a, cfg.n, cfg.b_deg, cfg.delta_s))


def test_geometry_matches_oracle(lib, port):
    from paper_2503_03479_b200 import api
    rng = np.random.default_rng(7)
    for _ in range(300):
        p = api.AffineParams(rng.uniform(-math.pi, math.pi), rng.uniform(1, 8), rng.uniform(0, math.pi),
                             rng.uniform(0.2, 4), rng.uniform(-40, 40), rng.uniform(-40, 40))
        s = api.simulation_from_params(p)
        assert np.array_equal(s, port.simulation_from_params(p.as_tuple()))
        a = api.affine_from_params(p)
        assert np.array_equal(a, port.affine_from_params(p.as_tuple()))
        assert np.array_equal(api.invert(a), port.invert(a))


def test_frame_matches_oracle_exactly(lib, port):
    # output frame (warp.cpp:24-42) of every default grid view at several sizes
    for p in port.build_grid():
        m = port.simulation_from_params(p)
        for w, h in [(40, 30), (64, 48), (640, 480), (1024, 768)]:
            img = np.zeros((h, w), np.float32) if w * h < 5000 else None
            W, H, tx, ty = C.c_int(), C.c_int(), C.c_double(), C.c_double()
            fwd = np.zeros(9)
            mm = np.ascontiguousarray(m.reshape(-1))
            assert lib.xa_warp_frame(mm.ctypes.data_as(C.c_void_p), w, h, C.byref(W), C.byref(H),
                                     C.byref(tx), C.byref(ty), fwd.ctypes.data_as(C.c_void_p)) == 0
            if img is not None:
                oim, otx, oty, ofwd = port.warp(img, m, "nearest")
                assert (W.value, H.value) == (oim.shape[1], oim.shape[0])
                assert (tx.value, ty.value) == (otx, oty)
                assert np.array_equal(fwd.reshape(3, 3), ofwd)


def test_geometry_errors(lib):
    from paper_2503_03479_b200 import api
    with pytest.raises(api.GeometryError):
        api.simulation_from_params(api.AffineParams(tilt=0.5))
    with pytest.raises(api.GeometryError):
        api.affine_from_params(api.AffineParams(scale=0.0))
    with pytest.raises(api.GeometryError):
        api.invert(np.zeros((3, 3)))
    with pytest.raises(api.GeometryError):
        api.build_param_grid(api.GridConfig(a=1.0))
