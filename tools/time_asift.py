"""Wall time of the ASIFT baseline on the config-2 pair (XA_ASIFT_TIMING=1
prints the phases).

usage: python tools/time_asift.py [n_grid] [max_points]
"""
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

import paper_2503_03479_b200 as xa  # noqa: E402
from paper_2503_03479_b200 import synth  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 5
    mp = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
    a, b = synth.config2(seed=2)
    a, b = a.astype(np.float32), b.astype(np.float32)
    grid = xa.build_param_grid(xa.GridConfig(n=n))
    xa.asift_correspondences(a, b, grid, mp)
    for _ in range(2):
        t0 = time.perf_counter()
        m = xa.asift_correspondences(a, b, grid, mp)
        print(f"asift n={n} views={len(grid.entries)} mp={mp}: {1e3 * (time.perf_counter() - t0):.1f} ms, "
              f"{len(m)} correspondences", flush=True)


if __name__ == "__main__":
    main()
