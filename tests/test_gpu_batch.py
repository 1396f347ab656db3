"""Batched coarse_search over many image pairs (BASELINE config 5,
xa_coarse_search_batch): every pair of a batch must give exactly what the
single-pair path gives for it, whatever the chunking (pairs per chunk K,
remainder chunks), and the 1920x1080 config-5 pairs must match the oracle."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _pairs(n, seed=31):
    from paper_2503_03479_b200 import synth
    return [synth.config1(seed=seed + i) for i in range(n)]


@pytest.mark.parametrize("chunk", ["1", "2", "5"])
@pytest.mark.parametrize("mode", ["nearest", "lanczos"])
def test_batch_equals_single_pairs(xa, port, chunk, mode, monkeypatch):
    monkeypatch.setenv("XA_BATCH_PAIRS", chunk)
    pairs = _pairs(5)
    grid = port.build_grid(n=3)
    eng = xa.Engine(0)
    res = xa.coarse_search_batch([a for a, _ in pairs], [b for _, b in pairs], grid, 500, 0.8,
                                 warp_mode=mode, engine=eng)
    assert len(res) == 5
    for (a, b), r in zip(pairs, res):
        one = xa.coarse_search(a, b, grid, 500, 0.8, warp_mode=mode, engine=eng)
        assert [c for _, c in r.per_entry_counts] == [c for _, c in one.per_entry_counts]
        assert r.per_entry_keypoints == one.per_entry_keypoints
        assert r.best_index == one.best_index


def test_batch_device_graph_replay_is_stable(xa, port):
    """Repeated device calls replay one CUDA graph: identical counts each time,
    and equal to the host entry point."""
    import torch
    pairs = _pairs(3, seed=57)
    grid = xa.build_param_grid(xa.GridConfig(n=3))
    n = len(grid.entries)
    eng = xa.Engine(0)
    da = [torch.from_numpy(a).cuda() for a, _ in pairs]
    db = [torch.from_numpy(b).cuda() for _, b in pairs]
    cnt = torch.zeros(3 * n, dtype=torch.int32, device="cuda")
    kpc = torch.zeros(3 * n, dtype=torch.int32, device="cuda")
    h, w = pairs[0][0].shape
    outs = []
    for _ in range(3):
        eng.coarse_search_batch_device(0, [t.data_ptr() for t in da], w, h, [t.data_ptr() for t in db],
                                       w, h, grid, 500, 0.8, 1, cnt.data_ptr(), kpc.data_ptr(),
                                       eng.stream)
        eng.check()
        outs.append((cnt.cpu().numpy().copy(), kpc.cpu().numpy().copy()))
    for o in outs[1:]:
        assert np.array_equal(o[0], outs[0][0]) and np.array_equal(o[1], outs[0][1])
    res = xa.coarse_search_batch([a for a, _ in pairs], [b for _, b in pairs], grid, 500, 0.8,
                                 warp_mode="lanczos", engine=eng)
    got = np.array([[c for _, c in r.per_entry_counts] for r in res]).reshape(-1)
    assert np.array_equal(got, outs[0][0])


def test_batch_rejects_mixed_sizes(xa, port):
    a, b = _pairs(1)[0]
    with pytest.raises(ValueError):
        xa.coarse_search_batch([a, a[:, :-8].copy()], [b, b], port.build_grid(n=2), 100)


def test_config5_batch_pairs_vs_single(xa, port):
    """8 of the 64 config-5 pairs (1920x1080, 43 views, 2000 kp, ratio 0.8,
    Lanczos): batched counts equal the single-pair path exactly."""
    from paper_2503_03479_b200 import synth
    pairs = synth.config5_pairs(list(range(0, 64, 8)))
    grid = xa.build_param_grid(xa.GridConfig())
    eng = xa.Engine(0)
    res = xa.coarse_search_batch([a for a, _ in pairs], [b for _, b in pairs], grid, 2000, 0.8,
                                 warp_mode="lanczos", engine=eng)
    for (a, b), r in zip(pairs, res):
        one = xa.coarse_search(a, b, grid, 2000, 0.8, warp_mode="lanczos", engine=eng)
        assert [c for _, c in r.per_entry_counts] == [c for _, c in one.per_entry_counts]
        assert r.per_entry_keypoints == one.per_entry_keypoints
        assert min(r.per_entry_keypoints) > 0


def test_batch_zero_background_under_poison(xa, port):
    """Chunks of one call reuse the pyramid slots; the zero background (band
    blocks whose sources are all outside the content, Lanczos tiles outside
    it) is written once per call, before the first chunk. With the pyramid
    pre-filled with a high-contrast pattern (XA_POISON_PYR) and 2 pairs per
    chunk (5 pairs: chunks of 2, 2, 1), every count equals the default run."""
    import json
    import subprocess
    import sys
    pairs = _pairs(5, seed=41)
    grid = port.build_grid(n=3)
    eng = xa.Engine(0)
    res = xa.coarse_search_batch([a for a, _ in pairs], [b for _, b in pairs], grid, 500, 0.8,
                                 warp_mode="lanczos", engine=eng)
    mine = [[c for _, c in r.per_entry_counts] for r in res]
    eng.close()
    code = (
        "import json, sys; sys.path.insert(0, '.')\n"
        "import paper_2503_03479_b200 as xa\n"
        "from paper_2503_03479_b200 import synth\n"
        "from oracle.oracle import Oracle\n"
        "pairs = [synth.config1(seed=41 + i) for i in range(5)]\n"
        "grid = Oracle('port').build_grid(n=3)\n"
        "res = xa.coarse_search_batch([a for a, _ in pairs], [b for _, b in pairs], grid, 500, 0.8,"
        " warp_mode='lanczos', engine=xa.Engine(0))\n"
        "print(json.dumps([[int(c) for _, c in r.per_entry_counts] for r in res]))\n")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True, text=True,
                         env=dict(os.environ, XA_POISON_PYR="1", XA_BATCH_PAIRS="2"), timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    assert json.loads(out.stdout.strip().splitlines()[-1]) == mine
