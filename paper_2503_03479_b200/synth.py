"""Seeded synthetic inputs with BASELINE.json's shapes.

The reference's published evaluation uses public image datasets that are not
in this container; these generators stand in for them. Both benchmark arms and
the tests use the same uint8 images.

Texture (BASELINE.json configs): a continuous scene of Gaussian blobs (sigma
U(2, 20) px, signed amplitude) and filled rectangles / ellipses at random
intensity over a mid-grey background, 200 blobs and 50 shapes per nominal
image area. A view of the scene under an affine camera map is rendered
analytically for the blobs (covariance pushed through the map plus a 0.5 px
pixel footprint) and with 4x4 supersampling for the shapes, then N(0, 5) noise
is added and the result is rounded and clipped to uint8. Rendering the views
this way gives band-limited tilted images without running any resampler from
the path under test.
"""
from __future__ import annotations

import dataclasses
import math
from typing import Tuple

import numpy as np


@dataclasses.dataclass
class Scene:
    width: float
    height: float
    blobs: np.ndarray   # (n, 4): cx, cy, sigma, amplitude
    shapes: np.ndarray  # (m, 7): kind (0 rect, 1 ellipse), cx, cy, a, b, angle, value
    background: float = 128.0


def make_scene(width: float, height: float, seed: int, nominal: Tuple[int, int] = None) -> Scene:
    """Scene over [0,width]x[0,height]; counts scale with area / nominal image area."""
    rng = np.random.default_rng(seed)
    nw, nh = nominal or (width, height)
    f = max(1.0, (width * height) / float(nw * nh))
    nb, ns = int(round(200 * f)), int(round(50 * f))
    blobs = np.stack([rng.uniform(0, width, nb), rng.uniform(0, height, nb),
                      rng.uniform(2.0, 20.0, nb),
                      rng.uniform(40.0, 110.0, nb) * rng.choice([-1.0, 1.0], nb)], 1)
    side = min(nw, nh)
    shapes = np.stack([rng.integers(0, 2, ns).astype(np.float64), rng.uniform(0, width, ns),
                       rng.uniform(0, height, ns), rng.uniform(side / 80, side / 10, ns),
                       rng.uniform(side / 80, side / 10, ns), rng.uniform(0, math.pi, ns),
                       rng.uniform(0, 255, ns)], 1)
    return Scene(float(width), float(height), blobs, shapes)


def view_map(tilt: float = 1.0, phi: float = 0.0, psi: float = 0.0, scale: float = 1.0) -> np.ndarray:
    """Linear camera map R(psi) S(scale) diag(1/tilt, 1) R(phi) (the reference's
    simulation_from_params, geometry.cpp:51-58, without translation)."""
    def rot(a):
        c, s = math.cos(a), math.sin(a)
        return np.array([[c, -s], [s, c]])
    return rot(psi) @ (scale * np.eye(2)) @ np.diag([1.0 / tilt, 1.0]) @ rot(phi)


def render(scene: Scene, lin: np.ndarray, out_w: int, out_h: int, noise_seed: int,
           noise_sigma: float = 5.0, center=None, ss: int = 4) -> np.ndarray:
    """uint8 image of the scene through x_img = lin @ (x_tex - c) + c_img."""
    lin = np.asarray(lin, np.float64)
    inv = np.linalg.inv(lin)
    c_tex = np.array(center if center is not None else (scene.width / 2, scene.height / 2))
    c_img = np.array([out_w / 2.0, out_h / 2.0])
    img = np.full((out_h, out_w), scene.background, np.float64)
    # blobs: Gaussian pushed through the map, plus the pixel footprint
    pix = 0.25 * np.eye(2)
    for cx, cy, sg, amp in scene.blobs:
        mu = lin @ (np.array([cx, cy]) - c_tex) + c_img
        cov0 = sg * sg * (lin @ lin.T)
        cov = cov0 + pix
        r = 3.5 * math.sqrt(max(cov[0, 0], cov[1, 1]))
        x0, x1 = int(max(0, mu[0] - r)), int(min(out_w - 1, mu[0] + r))
        y0, y1 = int(max(0, mu[1] - r)), int(min(out_h - 1, mu[1] + r))
        if x0 > x1 or y0 > y1:
            continue
        ic = np.linalg.inv(cov)
        gain = amp * math.sqrt(np.linalg.det(cov0) / np.linalg.det(cov))
        xs = np.arange(x0, x1 + 1) - mu[0]
        ys = np.arange(y0, y1 + 1)[:, None] - mu[1]
        q = ic[0, 0] * xs * xs + 2 * ic[0, 1] * xs * ys + ic[1, 1] * ys * ys
        img[y0:y1 + 1, x0:x1 + 1] += gain * np.exp(-0.5 * q)
    # shapes: 4x4 supersampled coverage, painted over
    sub = (np.arange(ss) + 0.5) / ss - 0.5
    for kind, cx, cy, a, b, ang, val in scene.shapes:
        corners = np.array([[-a, -b], [a, -b], [-a, b], [a, b]])
        ca, sa = math.cos(ang), math.sin(ang)
        rot = np.array([[ca, -sa], [sa, ca]])
        pts = (rot @ corners.T).T + [cx, cy]
        ip = (lin @ (pts - c_tex).T).T + c_img
        x0, x1 = int(max(0, ip[:, 0].min() - 1)), int(min(out_w - 1, ip[:, 0].max() + 1))
        y0, y1 = int(max(0, ip[:, 1].min() - 1)), int(min(out_h - 1, ip[:, 1].max() + 1))
        if x0 > x1 or y0 > y1:
            continue
        gx = (np.arange(x0, x1 + 1)[None, :, None, None] + sub[None, None, None, :])
        gy = (np.arange(y0, y1 + 1)[:, None, None, None] + sub[None, None, :, None])
        px = gx - c_img[0]
        py = gy - c_img[1]
        tx = inv[0, 0] * px + inv[0, 1] * py + c_tex[0] - cx
        ty = inv[1, 0] * px + inv[1, 1] * py + c_tex[1] - cy
        lx = tx * ca + ty * sa
        ly = -tx * sa + ty * ca
        if kind == 0:
            inside = (np.abs(lx) <= a) & (np.abs(ly) <= b)
        else:
            inside = (lx / a) ** 2 + (ly / b) ** 2 <= 1.0
        cov = inside.mean(axis=(2, 3))
        blk = img[y0:y1 + 1, x0:x1 + 1]
        img[y0:y1 + 1, x0:x1 + 1] = blk * (1 - cov) + val * cov
    rng = np.random.default_rng(noise_seed)
    img += rng.normal(0.0, noise_sigma, img.shape)
    return np.clip(np.rint(img), 0, 255).astype(np.uint8)


def texture(w: int, h: int, seed: int, ss: int = 4) -> np.ndarray:
    """Frontal w x h texture T(w, h, seed) of BASELINE.json."""
    return render(make_scene(w, h, seed), np.eye(2), w, h, noise_seed=seed + 1, ss=ss)


def pair(w: int, h: int, seed: int, view1=(1.0, 0.0, 0.0), view2=(2.0, 0.0, math.radians(30))):
    """Two w x h views (tilt, phi, psi) of one scene large enough to cover both footprints."""
    m1, m2 = view_map(*view1), view_map(*view2)
    ext = 0.0
    for m in (m1, m2):
        inv = np.linalg.inv(m)
        c = np.array([[-w / 2, -h / 2], [w / 2, -h / 2], [-w / 2, h / 2], [w / 2, h / 2]])
        ext = max(ext, float(np.abs((inv @ c.T)).max()))
    side = 2 * ext + 64
    scene = make_scene(side, side, seed, nominal=(w, h))
    return (render(scene, m1, w, h, noise_seed=seed + 11),
            render(scene, m2, w, h, noise_seed=seed + 12))


# ------------------------------------------------------------------ configs

def config1(seed: int = 1):
    """640x480 pair: reference frontal, second at absolute tilt t=2 (60 deg), rotation 30 deg."""
    return pair(640, 480, seed, (1.0, 0.0, 0.0), (2.0, 0.0, math.radians(30)))


def config2(seed: int = 2):
    """1024x768 pair at transition tilt: t1=4 at phi 0 vs t2=4*sqrt2 at phi 90 deg."""
    return pair(1024, 768, seed, (4.0, 0.0, 0.0), (4.0 * math.sqrt(2.0), math.pi / 2, 0.0))


def config3(seed: int = 3, size: int = 4096):
    """4096^2 texture for the view-simulation microbenchmark (2x2 shape supersampling)."""
    return texture(size, size, seed, ss=2)


T_MAX = 1.0 / math.cos(math.radians(80.0))  # absolute tilt 80 deg


def transition_tilt(view1, view2) -> float:
    """Transition tilt between two views (tilt, phi, psi): the singular-value
    ratio of the map image 1 -> image 2, view_map(view2) @ inv(view_map(view1))."""
    b = view_map(*view2) @ np.linalg.inv(view_map(*view1))
    sv = np.linalg.svd(b, compute_uv=False)
    return float(sv[0] / sv[1])


def config5_views(i: int, seed: int = 5):
    """Camera draws of config-5 pair i (BASELINE.json configs[4]): image 2 has
    absolute tilt U(0, 80 deg), in-plane rotation psi2 U(0, 360 deg) and tilt
    direction phi2 U(0, 180 deg); the transition tilt between the pair is drawn
    independently, tau = 1/cos(U(0, 90 deg)). Image 1 is then a view whose
    absolute tilt t1 (also within 0-80 deg) and tilt direction realise tau:
    t1 uniform over the values that can reach tau, the direction difference
    solved by bisection (tau grows monotonically from max(t1/t2, t2/t1) at 0 deg
    to t1*t2 at 90 deg). A tau beyond T_MAX * t2 (image 1 would need more than
    80 deg) is clamped to it. Returns (view1, view2, tau)."""
    rng = np.random.default_rng(seed * 1000 + i)
    t2 = 1.0 / math.cos(math.radians(rng.uniform(0.0, 80.0)))
    phi2, psi2 = rng.uniform(0, math.pi), rng.uniform(0, 2 * math.pi)
    tau = 1.0 / math.cos(math.radians(rng.uniform(0.0, 90.0)))
    tau = min(tau, T_MAX * t2)
    lo_t1 = max(1.0, tau / t2, t2 / tau)
    hi_t1 = min(T_MAX, tau * t2)
    t1 = rng.uniform(lo_t1, max(lo_t1, hi_t1))
    phi1 = rng.uniform(0, math.pi)

    def tt(d):
        return transition_tilt((t1, phi1, 0.0), (t2, phi1 + d, psi2))
    lo, hi = 0.0, math.pi / 2
    for _ in range(60):
        mid = 0.5 * (lo + hi)
        if tt(mid) < tau:
            lo = mid
        else:
            hi = mid
    d = 0.5 * (lo + hi)
    v1, v2 = (t1, phi1, 0.0), (t2, phi1 + d, psi2)
    return v1, v2, transition_tilt(v1, v2)


def config5_pair(i: int, seed: int = 5, w: int = 1920, h: int = 1080):
    """Pair i of BASELINE config 5: two w x h views of one scene (config5_views)."""
    v1, v2, _ = config5_views(i, seed)
    return pair(w, h, seed * 1000 + i, v1, v2)


def config5_pairs(indices=64, seed: int = 5, workers: int = None):
    """Pairs of config 5 (an int n means pairs 0..n-1), rendered in parallel
    processes (about 1.4 s each)."""
    import concurrent.futures as cf
    import os
    idx = list(range(indices)) if isinstance(indices, int) else list(indices)
    workers = workers or min(len(idx), os.cpu_count() or 1)
    if workers <= 1:
        return [config5_pair(i, seed) for i in idx]
    with cf.ProcessPoolExecutor(workers) as ex:
        return list(ex.map(config5_pair, idx, [seed] * len(idx)))


def descriptors(n: int, seed: int) -> np.ndarray:
    """n uniform random 256-bit descriptors as (n, 4) uint64."""
    rng = np.random.default_rng(seed)
    return rng.integers(0, np.iinfo(np.uint64).max, size=(n, 4), dtype=np.uint64, endpoint=True)


def config4(n: int = 200_000, seed: int = 4, planted: float = 0.2, max_flips: int = 40):
    """Query/train sets; `planted` of the queries are a train descriptor with
    U{0..max_flips} random bit flips. Returns (queries, train, planted_idx, src_idx)."""
    rng = np.random.default_rng(seed)
    train = descriptors(n, seed + 1)
    q = descriptors(n, seed + 2)
    k = int(n * planted)
    qi = rng.choice(n, k, replace=False)
    src = rng.integers(0, n, k)
    q[qi] = train[src]
    flips = rng.integers(0, max_flips + 1, k)
    bits = q.view(np.uint8).reshape(n, 32)
    for j, (row, nf) in enumerate(zip(qi, flips)):
        pos = rng.choice(256, nf, replace=False)
        np.bitwise_xor.at(bits[row], pos >> 3, (1 << (pos & 7)).astype(np.uint8))
    return q, train, qi, src
