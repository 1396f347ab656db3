"""A/B timing of the config-2 coarse step (graph replay, no stage events).

usage: python tools/time_coarse.py [steps]
"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2503_03479_b200 as xa  # noqa: E402
from paper_2503_03479_b200 import synth  # noqa: E402


def main():
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 50
    a, b = synth.config2(seed=2)
    grid = xa.build_param_grid(xa.GridConfig())
    n = len(grid.entries)
    eng = xa.Engine(0)
    dev = torch.device("cuda:0")
    stream = torch.cuda.ExternalStream(eng.stream, device=dev)
    da, db = torch.from_numpy(a).to(dev), torch.from_numpy(b).to(dev)
    counts = torch.zeros(n, dtype=torch.int32, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    h, w = a.shape

    def step():
        eng.coarse_search_device(0, da.data_ptr(), w, h, db.data_ptr(), b.shape[1], b.shape[0], grid,
                                 1000, 0.8, 1, counts.data_ptr(), 0, stream.cuda_stream)

    for _ in range(5):
        step()
    eng.check()
    ref = counts.cpu().numpy().copy()
    ts = []
    for k in range(steps):
        with torch.cuda.stream(stream):
            flush.fill_(k & 0xFF)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        step()
        e1.record(stream)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    assert np.array_equal(counts.cpu().numpy(), ref)
    print(f"ms/step median {np.median(ts):.4f} mean {np.mean(ts):.4f} min {np.min(ts):.4f}  counts sum {int(ref.sum())}")


if __name__ == "__main__":
    main()
