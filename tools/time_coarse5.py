"""Per-stage device times (CUDA events in the graph) of a config-5 coarse step
on P pairs (default 8 = one chunk), plus a digest of the per-entry counts so
A/B variants can be compared for identical results.

usage: python tools/time_coarse5.py [--pairs 8] [--steps 5] [--mode lanczos|nearest] [--once]
       (--once: a single un-profiled call, for ncu)
       XA_LIB_PATH=build/variants/NAME.so python tools/time_coarse5.py
"""
import argparse
import hashlib
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2503_03479_b200 as xa  # noqa: E402
from paper_2503_03479_b200 import synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--pairs", type=int, default=8)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--mode", default="lanczos")
    ap.add_argument("--once", action="store_true")
    ap.add_argument("--noprof", action="store_true", help="time the product graph (no stage events)")
    args = ap.parse_args()
    pairs = synth.config5_pairs(args.pairs)
    grid = xa.build_param_grid(xa.GridConfig())
    n = len(grid.entries)
    eng = xa.Engine(0)
    dev = torch.device("cuda:0")
    stream = torch.cuda.ExternalStream(eng.stream, device=dev)
    da = [torch.from_numpy(a).to(dev) for a, _ in pairs]
    db = [torch.from_numpy(b).to(dev) for _, b in pairs]
    P = len(pairs)
    counts = torch.zeros(P * n, dtype=torch.int32, device=dev)
    kpc = torch.zeros(P * n, dtype=torch.int32, device=dev)
    h, w = pairs[0][0].shape
    mode = 1 if args.mode == "lanczos" else 0

    def run():
        eng.coarse_search_batch_device(0, [t.data_ptr() for t in da], w, h, [t.data_ptr() for t in db], w, h,
                                       grid, 2000, 0.8, mode, counts.data_ptr(), kpc.data_ptr(),
                                       stream.cuda_stream)

    if args.once:
        run()
        torch.cuda.synchronize()
        eng.check()
        return
    for _ in range(2):
        run()
    eng.set_profiling(not args.noprof)
    tot = {}
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    run()
    torch.cuda.synchronize()
    wall = 0.0
    for k in range(args.steps):
        e0.record(stream)
        run()
        e1.record(stream)
        e1.synchronize()
        wall += e0.elapsed_time(e1)
        for name, ms in eng.stage_times():
            tot[name] = tot.get(name, 0.0) + ms
    eng.check()
    c = counts.cpu().numpy()
    print(json.dumps({"pairs": P, "mode": args.mode, "ms_step": round(wall / args.steps, 3),
                      "stages": {k: round(v / args.steps, 3) for k, v in tot.items()},
                      "counts_sha16": hashlib.sha256(c.tobytes()).hexdigest()[:16],
                      "sum_counts": int(c.sum()), "kp": int(kpc.sum().item())}))


if __name__ == "__main__":
    main()
