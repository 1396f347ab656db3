"""Generate tests/golden/golden.npz from the REFERENCE itself.

Runs the reference library compiled from /root/reference/proj/src by
oracle/Makefile (oracle/_ref/libxaref.so) on small seeded inputs and stores its
outputs. The fixtures pin the C restatement (tests/test_oracle.py) and, on the
GPU box where /root/reference does not exist, the CUDA path's parity chain.
Inputs use the reference tests' own generators (make_texture,
make_checkerboard, random_descriptors with std::mt19937_64) and seeds.

    make -C oracle && python tools/make_golden.py
"""
import hashlib
import math
import pathlib
import sys

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

from _mt64 import MT64, random_descriptors  # noqa: E402
from oracle.oracle import Oracle  # noqa: E402


def h(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main():
    rng = MT64(5489)
    for _ in range(9999):
        rng()
    assert rng() == 9981545732273789042, "mt19937_64 restatement broken"
    R = Oracle("reference")
    g = {}
    g["pattern_checksum"] = np.array([R.pattern_checksum()], np.uint64)
    g["pattern"] = R.pattern()
    g["texture_64x48_s3"] = R.make_texture(64, 48, 3)
    for w, hh, s in [(128, 128, 8), (200, 160, 9), (256, 256, 15), (31, 31, 7)]:
        g[f"texture_hash_{w}x{hh}_s{s}"] = np.frombuffer(
            bytes.fromhex(h(R.make_texture(w, hh, s))), np.uint8)
    g["grid_default"] = R.build_grid()
    g["grid_n3"] = R.build_grid(n=3)
    g["grid_ds0"] = R.build_grid(delta_s=0.0)
    img = R.make_texture(48, 40, 5)
    g["aa_in"] = img
    for name, (t, phi) in {"aa_t2_phi0": (2.0, 0.0), "aa_t2_phi06": (2.0, 0.6),
                           "aa_t4s2_phi1": (4 * math.sqrt(2), 1.1)}.items():
        g[name] = R.antialias_tilt(img, t, phi)
    small = R.make_texture(40, 30, 9)
    g["warp_in"] = small
    mats = {
        "rot90": np.array([[0, -1, 0], [1, 0, 0], [0, 0, 1]], np.float64),
        "stretch2": np.diag([2.0, 1.0, 1.0]),
        "sim_t2_phi36_s2": R.simulation_from_params([0, 2.0, math.radians(36), 2.0, 0, 0]),
        "sim_t28_phi1_s15": R.simulation_from_params([0.3, 2 * math.sqrt(2), 1.0, 1.5, 0, 0]),
    }
    for mname, m in mats.items():
        g[f"mat_{mname}"] = m
        for mode in ("nearest", "lanczos"):
            im, tx, ty, fwd = R.warp(small, m, mode)
            g[f"warp_{mode}_{mname}"] = im
            g[f"warp_{mode}_{mname}_frame"] = np.array([tx, ty, *fwd.reshape(-1)])
    # synth_warp_case (eval.cpp:101-141): projective Lanczos renders of the
    # harness, one mild and one strong perspective homography
    g["synth_in"] = R.make_texture(56, 44, 4)
    for hname, hm in {"synth_mild": [[0.92, 0.12, 3.0], [-0.08, 1.04, -2.0], [3e-4, -2e-4, 1.0]],
                      "synth_strong": [[0.7, -0.5, 10.0], [0.45, 0.8, -4.0], [2.5e-3, 1.5e-3, 1.0]]
                      }.items():
        hm = np.array(hm, np.float64)
        im, comp = R.synth_warp_case(g["synth_in"], hm)
        g[f"{hname}_h"], g[hname], g[f"{hname}_composed"] = hm, im, comp
    # ORB on the reference tests' images
    tex = R.make_texture(128, 128, 8)
    kps = R.detect(tex, 200)
    g["orb_tex128_kps"] = kps
    k2, d2 = R.describe(tex, kps)
    g["orb_tex128_desc_kps"] = k2
    g["orb_tex128_desc"] = d2
    cb = R.make_checkerboard(256, 256, 32)
    kc = R.detect(cb, 1000)
    g["orb_checker_kps"] = kc
    g["orb_checker_desc"] = R.describe(cb, kc)[1]
    t256 = R.make_texture(256, 256, 15)
    g["orb_tex256_kps_all"] = R.detect(t256, 1000)
    g["orb_tex256_kps_cap50"] = R.detect(t256, 50)
    relax = R.make_texture(200, 200, 21) * np.float32(0.12) + np.float32(90)
    g["orb_relax_in_hash"] = np.frombuffer(bytes.fromhex(h(relax)), np.uint8)
    g["orb_relax_kps"] = R.detect(relax, 1000)
    # matcher KATs (test_features_binary.cpp:233-246, acceptance_main.cpp:314-350)
    da, db = random_descriptors(500, 101), random_descriptors(500, 202)
    g["desc_s101"], g["desc_s202"] = da, db
    for r in (0.6, 0.75, 0.9, 1.0):
        g[f"match_s101_s202_r{r}"] = R.match(da, db, r)
    rng = MT64(161)
    acc = np.array([[rng() for _ in range(4)] for _ in range(1000)], np.uint64)
    g["desc_s161_a"], g["desc_s161_b"] = acc[:500], acc[500:]
    g["match_s161_r0.75"] = R.match(acc[:500], acc[500:], 0.75)
    g["match_s161_r0.6"] = R.match(acc[:500], acc[500:], 0.6)
    # coarse search (test_pipeline.cpp:172-205 style, small)
    ct = R.make_texture(128, 128, 19)
    p = [0, math.sqrt(2), 0.4, 1, 0, 0]
    filt = R.antialias_tilt(ct, p[1], p[2])
    tgt = R.warp(filt, R.simulation_from_params(p), "nearest")[0]
    grid = R.build_grid(n=2)
    g["coarse_in"], g["coarse_tgt"], g["coarse_grid"] = ct, tgt, grid
    for mode in ("nearest", "lanczos"):
        c, kpc, best = R.coarse_search(ct, tgt, grid, 300, 0.75, mode, threads=4)
        g[f"coarse_{mode}_counts"] = c
        g[f"coarse_{mode}_best"] = np.array([best])
    out = ROOT / "tests" / "golden" / "golden.npz"
    out.parent.mkdir(parents=True, exist_ok=True)
    np.savez_compressed(out, **g)
    print("wrote", out, out.stat().st_size, "bytes,", len(g), "arrays")


if __name__ == "__main__":
    main()
