"""GPU Hamming matcher bit-exact against the oracle and the reference's
matcher tests (proj/tests/test_features_binary.cpp:190-282,
acceptance_main.cpp:314-350), at test sizes and at BASELINE config-4 size."""
import numpy as np
import pytest

from _mt64 import random_descriptors

pytestmark = pytest.mark.gpu


def arr(m):
    return np.stack([m["idx_a"], m["idx_b"], m["distance"].astype(np.int32)], 1) if len(m) else \
        np.zeros((0, 3), np.int32)


@pytest.mark.parametrize("r", [0.6, 0.75, 0.9, 1.0])
def test_golden_500x500(xa, golden, r):
    got = xa.match_hamming(golden["desc_s101"], golden["desc_s202"], r)
    assert np.array_equal(arr(got), golden[f"match_s101_s202_r{r}"])


def test_golden_acceptance(xa, golden):
    a, b = golden["desc_s161_a"], golden["desc_s161_b"]
    assert np.array_equal(arr(xa.match_hamming(a, b, 0.75)), golden["match_s161_r0.75"])
    assert np.array_equal(arr(xa.match_hamming(a, b, 0.6)), golden["match_s161_r0.6"])


def test_self_match_identity(xa):
    d = random_descriptors(64, 3)
    m = xa.match_hamming(d, d, 0.75)
    assert len(m) == 64
    assert np.array_equal(m["idx_a"], np.arange(64)) and np.array_equal(m["idx_b"], np.arange(64))
    assert np.all(m["distance"] == 0)


def test_single_candidate_rule(xa):
    a = random_descriptors(1, 9)
    b = a.copy()
    bits = b.view(np.uint8).reshape(-1)
    for i in range(100):
        b[0, i >> 6] ^= np.uint64(1) << np.uint64(i & 63)
    assert len(xa.match_hamming(a, b, 0.75)) == 1
    for i in range(100, 200):
        b[0, i >> 6] ^= np.uint64(1) << np.uint64(i & 63)
    assert len(xa.match_hamming(a, b, 0.75)) == 0
    del bits


def test_empty(xa):
    assert len(xa.match_hamming(np.zeros((0, 4), np.uint64), random_descriptors(5, 1), 0.75)) == 0
    assert len(xa.match_hamming(random_descriptors(5, 1), np.zeros((0, 4), np.uint64), 0.75)) == 0


def test_ties_and_duplicates(xa, port):
    # duplicated train rows: lowest index wins and second == best (orb.cpp:259-265)
    rng = np.random.default_rng(0)
    b = random_descriptors(300, 5)
    b = np.vstack([b, b[::3], b[:50]])
    a = np.vstack([b[rng.integers(0, len(b), 200)], random_descriptors(100, 6)])
    for r in (0.5, 0.8, 1.0):
        assert np.array_equal(arr(xa.match_hamming(a, b, r)), port.match(a, b, r))


def test_permutation_relabels(xa):
    da, db = random_descriptors(120, 31), random_descriptors(120, 41)
    base = xa.match_hamming(da, db, 0.8)
    perm = np.arange(119, -1, -1)
    db2 = np.empty_like(db)
    db2[perm] = db
    p = xa.match_hamming(da, db2, 0.8)
    assert np.array_equal(base["idx_a"], p["idx_a"])
    assert np.array_equal(perm[base["idx_b"]], p["idx_b"])


@pytest.mark.parametrize("na,nb", [(1, 1), (3, 2000), (5000, 7), (4096, 4096), (20000, 30000)])
def test_random_sizes_vs_oracle(xa, port, na, nb):
    from paper_2503_03479_b200 import synth
    a, b = synth.descriptors(na, na), synth.descriptors(nb, nb + 1)
    # plant near-duplicates so the ratio test passes often
    k = min(na, nb) // 3
    a[:k] = b[:k]
    a[:k, 0] ^= np.uint64(0xFF)
    for r in (0.8,):
        assert np.array_equal(arr(xa.match_hamming(a, b, r)), port.match(a, b, r))


def test_config4_full_size_properties(xa, port):
    """BASELINE config 4 (200k x 200k): full-size run checked by properties and
    exactly against the oracle's match_hamming over every query."""
    import torch
    from paper_2503_03479_b200 import synth
    q, t, qi, src = synth.config4(200_000)
    eng = xa.Engine(0)
    dq, dt = torch.from_numpy(q.view(np.int64)).cuda(), torch.from_numpy(t.view(np.int64)).cuda()
    n = len(q)
    bi = torch.empty(n, dtype=torch.int32, device="cuda")
    bd = torch.empty(n, dtype=torch.int16, device="cuda")
    sd = torch.empty(n, dtype=torch.int16, device="cuda")
    cnt = torch.zeros(1, dtype=torch.int32, device="cuda")
    eng.match_hamming_device(dq.data_ptr(), n, dt.data_ptr(), n, 0.8, bi.data_ptr(), bd.data_ptr(),
                             sd.data_ptr(), cnt.data_ptr())
    torch.cuda.synchronize()
    bi, bd, sd = bi.cpu().numpy().view(np.uint32), bd.cpu().numpy(), sd.cpu().numpy()
    keep = bd < 0.8 * sd
    assert int(cnt.item()) == int(keep.sum())
    # planted queries with <= 40 flips recover their source (or an equal-distance earlier twin)
    x = np.bitwise_xor(q[qi], t[src])
    dist = np.unpackbits(x.view(np.uint8), axis=1).sum(1)
    assert np.all(bd[qi] <= dist)
    assert np.mean(bi[qi] == src) > 0.999
    # exact oracle agreement on ALL 200k queries against the full train set:
    # contiguous query shards on the host threads (match_hamming per shard,
    # idx_a offset), i.e. the reference's matcher over the whole query set
    import concurrent.futures as cf
    import os
    nt = os.cpu_count() or 1
    bounds = np.linspace(0, n, nt + 1).astype(int)

    def shard(k):
        lo, hi = bounds[k], bounds[k + 1]
        m = port.match(q[lo:hi], t, 0.8)
        m[:, 0] += lo
        return m
    with cf.ThreadPoolExecutor(nt) as ex:
        want = np.concatenate(list(ex.map(shard, range(nt))))
    got_i = np.nonzero(keep)[0]
    assert np.array_equal(want[:, 0], got_i)
    assert np.array_equal(want[:, 1], bi[got_i].astype(np.int32))
    assert np.array_equal(want[:, 2], bd[got_i].astype(np.int32))
    eng.close()
