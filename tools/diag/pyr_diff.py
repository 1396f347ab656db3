"""Check the device ORB pyramid (xa_engine_read_pyramid after a detect call)
against an exact numpy replay of build_pyramid (orb.cpp:130-141 +
image.cpp:51-70, float32 ops in the reference's order) on a crop of the
config-1 texture: per level, number of differing pixels and the first ones."""
import ctypes as C
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_2503_03479_b200 as xa  # noqa: E402
from paper_2503_03479_b200 import _lib, synth  # noqa: E402

f32 = np.float32


def levels(w, h):
    out = [(w, h)]
    for L in range(1, 8):
        sc = 1.2 ** L
        lw, lh = int(round(w / sc)), int(round(h / sc))
        if lw < 32 or lh < 32:
            break
        out.append((lw, lh))
    return out


def resize(img, w, h):
    H0, W0 = img.shape
    sx, sy = W0 / w, H0 / h
    fx = (np.arange(w) + 0.5) * sx - 0.5
    fy = (np.arange(h) + 0.5) * sy - 0.5
    x0, y0 = np.floor(fx).astype(int), np.floor(fy).astype(int)
    wx, wy = (fx - x0).astype(f32), (fy - y0).astype(f32)
    xa, xb = np.clip(x0, 0, W0 - 1), np.clip(x0 + 1, 0, W0 - 1)
    ya, yb = np.clip(y0, 0, H0 - 1), np.clip(y0 + 1, 0, H0 - 1)
    v00, v10 = img[ya][:, xa], img[ya][:, xb]
    v01, v11 = img[yb][:, xa], img[yb][:, xb]
    iwx, iwy = f32(1) - wx, (f32(1) - wy)[:, None]
    WY = wy[:, None]
    top = iwx * v00 + wx * v10
    bot = iwx * v01 + wx * v11
    return (iwy * top + WY * bot).astype(f32)


W = int(sys.argv[1]) if len(sys.argv) > 1 else 200
Hh = int(sys.argv[2]) if len(sys.argv) > 2 else 200
a, _ = synth.config1(seed=11)
a = np.ascontiguousarray(a[:Hh, :W]).astype(f32)
e = xa.Engine(0)
xa.detect_oriented_corners(a, 2000, engine=e)
lv = levels(W, Hh)
tot = sum(-(-((w + 3) // 4 * 4) * h // 32) * 32 for w, h in lv)
buf = np.zeros(tot, f32)
assert _lib.lib().xa_engine_read_pyramid(e.handle, buf.ctypes.data_as(C.c_void_p), tot) == 0
off = 0
for L, (w, h) in enumerate(lv):
    p = (w + 3) // 4 * 4
    got = buf[off:off + p * h].reshape(h, p)[:, :w]
    want = a if L == 0 else resize(a, w, h)
    d = np.argwhere(got != want)
    print(L, w, h, "ndiff", len(d), "maxabs", float(np.abs(got - want).max()), "first", d[:6].tolist())
    for r in np.unique(d[:, 0])[:6]:
        cs = d[d[:, 0] == r, 1]
        print("   row", r, "cols", cs.min(), "..", cs.max(), "n", len(cs), "got", got[r, cs[:3]], "want", want[r, cs[:3]])
    off += -(-p * h // 32) * 32
