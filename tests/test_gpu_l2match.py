"""GPU L2 ratio matcher (match_ratio, sift.cpp:388-418 — SURVEY.md §8f row 1's
matcher) bit-exact against the reference compiled from its sources and the C
restatement, on SIFT-like descriptors (non-negative, L2 norm 512) with planted
near-duplicates, exact duplicates and ties."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def sift_like(n, seed):
    rng = np.random.default_rng(seed)
    d = rng.gamma(0.6, 1.0, size=(n, 128)).astype(np.float32)
    d = np.minimum(d / np.linalg.norm(d, axis=1, keepdims=True), 0.2)
    return (512.0 * d / np.linalg.norm(d, axis=1, keepdims=True)).astype(np.float32)


def planted(na, nb, seed):
    rng = np.random.default_rng(seed)
    a, b = sift_like(na, seed), sift_like(nb, seed + 1)
    k = min(na, nb) // 3
    idx = rng.choice(nb, k, replace=False)
    b[idx] = a[:k] + rng.normal(0, 2.0, size=(k, 128)).astype(np.float32)  # near-duplicates
    if nb > 8:
        b[nb // 2] = b[nb // 2 + 1]  # an exact tie in B
        b[3] = a[min(5, na - 1)]     # an exact duplicate
    return a, b


def check(xa, orc, a, b, ratio):
    got = xa.match_ratio(a, b, ratio)
    want = orc.match_ratio(a, b, ratio)
    assert got.dtype.names == ("idx_a", "idx_b", "distance")
    assert np.array_equal(got["idx_a"], want["idx_a"])
    assert np.array_equal(got["idx_b"], want["idx_b"])
    assert np.array_equal(got["distance"].view(np.uint32), want["distance"].view(np.uint32))
    return len(got)


@pytest.mark.parametrize("na,nb,seed", [(300, 400, 1), (33, 1000, 2), (257, 65, 3), (1, 5, 4)])
@pytest.mark.parametrize("ratio", [0.6, 0.8, 1.0])
def test_vs_reference(xa, ref, na, nb, seed, ratio):
    a, b = planted(na, nb, seed)
    check(xa, ref, a, b, ratio)


def test_vs_port_larger(xa, port):
    a, b = planted(1500, 1200, 9)
    assert check(xa, port, a, b, 0.8) > 300


def test_edge_cases(xa, ref):
    a, b = planted(20, 20, 5)
    assert len(xa.match_ratio(a[:0], b, 0.75)) == 0
    assert len(xa.match_ratio(a, b[:0], 0.75)) == 0
    # single candidate: second missing -> distance 1024 (sift.cpp:414)
    check(xa, ref, a[:4], b[:1], 0.75)
    check(xa, ref, a, a, 0.75)  # self match: distance 0, identity
    m = xa.match_ratio(a, a, 0.75)
    assert np.array_equal(m["idx_a"], m["idx_b"]) and np.all(m["distance"] == 0)
