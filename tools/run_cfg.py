"""One device call of a secondary BASELINE workload (for ncu captures):
    python tools/run_cfg.py cfg3   # 4096^2 texture -> 43 Lanczos views (uint8)
    python tools/run_cfg.py cfg4   # 200k x 200k Hamming top-2 ratio matching
"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2503_03479_b200 as xa  # noqa: E402
from paper_2503_03479_b200 import synth  # noqa: E402


def main():
    which = sys.argv[1]
    eng = xa.Engine(0)
    if which == "cfg3":
        src = synth.config3()
        grid = xa.build_param_grid(xa.GridConfig(delta_s=0.0))
        _, _, _, total = eng.simulate_views_plan(4096, 4096, grid, 1)
        d_src = torch.from_numpy(src).cuda()
        d_out = torch.empty(total, dtype=torch.uint8, device="cuda")
        eng.simulate_views_device(d_src.data_ptr(), 4096, 4096, grid, 1, d_out.data_ptr())
    else:
        q, t, _, _ = synth.config4(200_000)
        n = len(q)
        dq, dt = torch.from_numpy(q.view(np.int64)).cuda(), torch.from_numpy(t.view(np.int64)).cuda()
        bi = torch.empty(n, dtype=torch.int32, device="cuda")
        bd = torch.empty(n, dtype=torch.int16, device="cuda")
        sd = torch.empty(n, dtype=torch.int16, device="cuda")
        cnt = torch.zeros(1, dtype=torch.int32, device="cuda")
        eng.match_hamming_device(dq.data_ptr(), n, dt.data_ptr(), n, 0.8, bi.data_ptr(), bd.data_ptr(),
                                 sd.data_ptr(), cnt.data_ptr())
    torch.cuda.synchronize()
    eng.check()


if __name__ == "__main__":
    main()
