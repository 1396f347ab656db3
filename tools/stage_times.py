"""Per-stage device times (CUDA events in the graph) of the config-2 coarse
step, without any result checks (for A/B variants that compute garbage).

usage: python tools/stage_times.py [steps]
"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2503_03479_b200 as xa  # noqa: E402
from paper_2503_03479_b200 import synth  # noqa: E402


def main():
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
    a, b = synth.config2(seed=2)
    grid = xa.build_param_grid(xa.GridConfig())
    n = len(grid.entries)
    eng = xa.Engine(0)
    dev = torch.device("cuda:0")
    stream = torch.cuda.ExternalStream(eng.stream, device=dev)
    da, db = torch.from_numpy(a).to(dev), torch.from_numpy(b).to(dev)
    counts = torch.zeros(n, dtype=torch.int32, device=dev)
    h, w = a.shape
    eng.set_profiling(True)
    tot = {}
    for k in range(steps + 3):
        eng.coarse_search_device(0, da.data_ptr(), w, h, db.data_ptr(), b.shape[1], b.shape[0], grid,
                                 1000, 0.8, 1, counts.data_ptr(), 0, stream.cuda_stream)
        st = eng.stage_times()
        if k >= 3:
            for name, ms in st:
                tot[name] = tot.get(name, 0.0) + ms
    print({k: round(v / steps, 4) for k, v in tot.items()})


if __name__ == "__main__":
    main()
