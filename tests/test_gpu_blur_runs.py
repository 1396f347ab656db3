"""The pipeline's directional blur as stencil runs (k_blur_runs, default) against
the per-cell stencil kernel (XA_BLUR_RUNS=0, read once per process: run in a
subprocess): the two sum the same float cells in different orders, so the
uint8 views of every grid entry (row-run and column-run stencils, tilts up to
4 sqrt 2, interior and border tiles) may differ only by one level at rounding
ties, on a vanishing fraction of pixels."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CODE = r"""
import sys
import numpy as np, torch
sys.path.insert(0, ".")
import paper_2503_03479_b200 as xa
from paper_2503_03479_b200 import synth
src, _ = synth.config2(seed=3)
h, w = src.shape
grid = xa.build_param_grid(xa.GridConfig())
eng = xa.Engine(0)
offs, ws, hs, total = eng.simulate_views_plan(w, h, grid, 1)
d_src = torch.from_numpy(np.ascontiguousarray(src)).cuda()
d_out = torch.empty(total, dtype=torch.uint8, device="cuda")
eng.simulate_views_device(d_src.data_ptr(), w, h, grid, 1, d_out.data_ptr())
torch.cuda.synchronize()
np.save(sys.argv[1], d_out.cpu().numpy())
"""


def views(path, **env):
    r = subprocess.run([sys.executable, "-c", CODE, path], cwd=ROOT, env=dict(os.environ, **env),
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    return np.load(path)


def test_blur_runs_match_stencil(tmp_path):
    a = views(str(tmp_path / "runs.npy")).astype(np.int16)
    b = views(str(tmp_path / "cells.npy"), XA_BLUR_RUNS="0").astype(np.int16)
    d = np.abs(a - b)
    assert d.max() <= 1
    assert np.count_nonzero(d) <= 1e-4 * d.size, np.count_nonzero(d)
