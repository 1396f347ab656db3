"""Multi-GPU sharding of config 5 on the device path. Only one
GPU is available here, so the sharding logic is exercised with several
independent engines / ranks on cuda:0 (their kernels never wait on one
another); results must be byte-identical to the single-engine batch."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _pairs(n, seed=71):
    from paper_2503_03479_b200 import synth
    return [synth.config1(seed=seed + i) for i in range(n)]


def _counts(res):
    return np.array([[c for _, c in r.per_entry_counts] for r in res])


def test_multi_engines_equal_batch(xa, port):
    pairs = _pairs(5)
    grid = port.build_grid(n=3)
    A, B = [a for a, _ in pairs], [b for _, b in pairs]
    one = xa.coarse_search_batch(A, B, grid, 500, 0.8, warp_mode="lanczos")
    for k in (1, 2, 3):
        engines = [xa.Engine(0) for _ in range(k)]
        got = xa.coarse_search_multi(A, B, grid, 500, 0.8, warp_mode="lanczos", engines=engines)
        assert np.array_equal(_counts(got), _counts(one))
        assert [r.best_index for r in got] == [r.best_index for r in one]
        assert [r.per_entry_keypoints for r in got] == [r.per_entry_keypoints for r in one]


def test_nccl_world1_equals_batch(xa, port):
    pairs = _pairs(3, seed=91)
    grid = port.build_grid(n=3)
    A, B = [a for a, _ in pairs], [b for _, b in pairs]
    one = xa.coarse_search_batch(A, B, grid, 500, 0.8, warp_mode="lanczos")
    comm = xa.api.nccl_comm_init(xa.api.nccl_unique_id(), 0, 1, 0)
    try:
        got = xa.coarse_search_nccl(A, B, grid, comm, 0, 1, 500, 0.8, warp_mode="lanczos")
    finally:
        xa.api.nccl_comm_destroy(comm)
    assert np.array_equal(_counts(got), _counts(one))
    assert [r.best_index for r in got] == [r.best_index for r in one]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK="0")
    import torch.distributed as dist
    import paper_2503_03479_b200 as xa
    from paper_2503_03479_b200 import dist as D
    r, w, _ = D.init_from_env(backend="gloo")
    pairs = _pairs(5)
    grid = xa.build_param_grid(xa.GridConfig(n=3))
    eng = xa.Engine(0)

    def run_block(lo, hi):
        res = xa.coarse_search_batch([a for a, _ in pairs[lo:hi]], [b for _, b in pairs[lo:hi]], grid,
                                     500, 0.8, warp_mode="lanczos", engine=eng)
        return _counts(res)
    counts, best = D.coarse_search_pairs_sharded(5, len(grid.entries), r, w, run_block)
    q.put((r, counts.tolist(), best))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(600)
def test_two_ranks_gloo_equal_one(xa, port):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = _free_port()
    procs = [ctx.Process(target=_rank, args=(r, 2, p, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = sorted(q.get(timeout=500) for _ in range(2))
    for pr in procs:
        pr.join(60)
        assert pr.exitcode == 0
    assert res[0][1:] == res[1][1:]
    pairs = _pairs(5)
    one = xa.coarse_search_batch([a for a, _ in pairs], [b for _, b in pairs],
                                 xa.build_param_grid(xa.GridConfig(n=3)), 500, 0.8, warp_mode="lanczos")
    assert res[0][1] == _counts(one).tolist()
    assert res[0][2] == [r.best_index for r in one]
