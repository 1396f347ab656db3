"""The three Hamming matcher implementations give identical outputs: tcgen05
kind::i8 (default), warp-level IMMA (XA_MATCH_UMMA=0) and XOR + POPC
(XA_MATCH_TC=0), on the large-set API (train slices + merge) and on the
coarse path (per-view jobs on real ORB descriptors). The switches are read
once per process, so each variant runs in its own interpreter."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

LARGE = r"""
import hashlib, json, sys
import numpy as np, torch
sys.path.insert(0, ".")
import paper_2503_03479_b200 as xa
from paper_2503_03479_b200 import synth
out = {}
for n_q, n_t in ((60000, 50000), (777, 129), (1, 5000)):
    q, t, _, _ = synth.config4(max(n_q, n_t))
    q, t = q[:n_q].copy(), t[:n_t].copy()
    t[: n_t // 7] = t[n_t // 2 : n_t // 2 + n_t // 7]   # duplicated train rows: index ties
    eng = xa.Engine(0)
    dq, dt = torch.from_numpy(q.view(np.int64)).cuda(), torch.from_numpy(t.view(np.int64)).cuda()
    bi = torch.empty(n_q, dtype=torch.int32, device="cuda")
    bd = torch.empty(n_q, dtype=torch.int16, device="cuda")
    sd = torch.empty(n_q, dtype=torch.int16, device="cuda")
    cnt = torch.zeros(1, dtype=torch.int32, device="cuda")
    eng.match_hamming_device(dq.data_ptr(), n_q, dt.data_ptr(), n_t, 0.8, bi.data_ptr(), bd.data_ptr(),
                             sd.data_ptr(), cnt.data_ptr())
    torch.cuda.synchronize()
    eng.check()
    h = hashlib.sha256()
    for x in (bi, bd, sd, cnt):
        h.update(x.cpu().numpy().tobytes())
    out[f"{n_q}x{n_t}"] = [h.hexdigest()[:16], int(cnt.item())]
print(json.dumps(out))
"""

COARSE = r"""
import json, sys
sys.path.insert(0, ".")
import paper_2503_03479_b200 as xa
from paper_2503_03479_b200 import synth
pairs = synth.config5_pairs(2)
grid = xa.build_param_grid(xa.GridConfig())
res = xa.coarse_search_batch([a for a, _ in pairs], [b for _, b in pairs], grid, 2000, 0.8, warp_mode="lanczos")
print(json.dumps([[c for _, c in r.per_entry_counts] for r in res]))
"""


def run(code, **env):
    e = dict(os.environ, **env)
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=e, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


def test_large_set_matchers_identical():
    umma = run(LARGE)
    assert run(LARGE, XA_MATCH_UMMA="0") == umma
    assert run(LARGE, XA_MATCH_TC="0") == umma


def test_coarse_matchers_identical():
    umma = run(COARSE)
    assert run(COARSE, XA_MATCH_UMMA="0") == umma
    assert run(COARSE, XA_MATCH_TC="0") == umma
