"""MT19937-64 (Matsumoto & Nishimura), matching std::mt19937_64, for the
reference tests' random_descriptors helper (proj/tests/test_features_binary.cpp:18-24:
every descriptor word is one raw draw)."""
import numpy as np

_N, _M = 312, 156
_MASK = (1 << 64) - 1


class MT64:
    def __init__(self, seed: int):
        self.mt = [0] * _N
        self.mt[0] = seed & _MASK
        for i in range(1, _N):
            prev = self.mt[i - 1]
            self.mt[i] = (6364136223846793005 * (prev ^ (prev >> 62)) + i) & _MASK
        self.i = _N

    def _twist(self):
        mt = self.mt
        for i in range(_N):
            x = (mt[i] & 0xFFFFFFFF80000000) | (mt[(i + 1) % _N] & 0x7FFFFFFF)
            xa = x >> 1
            if x & 1:
                xa ^= 0xB5026F5AA96619E9
            mt[i] = mt[(i + _M) % _N] ^ xa
        self.i = 0

    def __call__(self) -> int:
        if self.i >= _N:
            self._twist()
        y = self.mt[self.i]
        self.i += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000 & _MASK
        y ^= (y << 37) & 0xFFF7EEE000000000 & _MASK
        y ^= y >> 43
        return y & _MASK


def random_descriptors(n: int, seed: int) -> np.ndarray:
    rng = MT64(seed)
    return np.array([[rng() for _ in range(4)] for _ in range(n)], dtype=np.uint64).reshape(n, 4)
