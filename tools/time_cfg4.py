"""Config-4 Hamming matching timing (200k x 200k, device-resident inputs):
median of N calls by CUDA events + a digest of the outputs, so the tensor-core
matcher and the XOR + POPC one (XA_MATCH_TC=0) can be compared for identical
results.   python tools/time_cfg4.py [N]
"""
import hashlib
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2503_03479_b200 as xa  # noqa: E402
from paper_2503_03479_b200 import synth  # noqa: E402


def main():
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
    eng = xa.Engine(0)
    q, t, _, _ = synth.config4(200_000)
    n = len(q)
    dq, dt = torch.from_numpy(q.view(np.int64)).cuda(), torch.from_numpy(t.view(np.int64)).cuda()
    bi = torch.empty(n, dtype=torch.int32, device="cuda")
    bd = torch.empty(n, dtype=torch.int16, device="cuda")
    sd = torch.empty(n, dtype=torch.int16, device="cuda")
    cnt = torch.zeros(1, dtype=torch.int32, device="cuda")
    stream = torch.cuda.ExternalStream(eng.stream)

    def run():
        eng.match_hamming_device(dq.data_ptr(), n, dt.data_ptr(), n, 0.8, bi.data_ptr(), bd.data_ptr(),
                                 sd.data_ptr(), cnt.data_ptr())

    run()
    torch.cuda.synchronize()
    eng.check()
    ms = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        run()
        e1.record(stream)
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    h = hashlib.sha256()
    for x in (bi, bd, sd, cnt):
        h.update(x.cpu().numpy().tobytes())
    med = float(np.median(ms))
    print(json.dumps({"ms": med, "cmp_per_s": n * n / (med * 1e-3), "matches": int(cnt.item()),
                      "digest": h.hexdigest()[:16]}))


if __name__ == "__main__":
    main()
