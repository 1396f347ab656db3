"""Multi-GPU sharding of the hot path: one process per GPU.

The path is embarrassingly parallel; the only exchange is gathering results:

  * views   — grid entries of one pair are dealt to ranks by LPT on an
              estimated cost (output pixels x ORB work), each rank runs its
              entries through the batched coarse search, per-entry counts are
              all-gathered and every rank applies the reference's strict-'>'
              grid-order argmax (pipeline.cpp:142-150);
  * pairs   — whole image pairs are split into contiguous blocks, one per
              rank (BASELINE config 5); each rank runs its block through the
              batched device pipeline and the per-pair counts are all-gathered;
  * queries — Hamming matching splits the query set into contiguous blocks
              against a replicated train set; (best_idx, best, second) per
              query are all-gathered (BASELINE config 4).

Results are identical for any world size by construction (each unit is
independent and gathered in unit order). Collectives go through
torch.distributed: NCCL over NVLink on GPUs, gloo in the CPU tests.
"""
from __future__ import annotations

import math
import os
from typing import Callable, List, Sequence, Tuple

import numpy as np


def init_from_env(backend: str = None):
    """(rank, world, local_rank); initialises torch.distributed when WORLD_SIZE > 1."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        if not dist.is_initialized():
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            if backend is None:
                # XA_DIST_BACKEND=gloo runs the multi-rank host logic with CPU
                # collectives (e.g. to exercise it with fewer GPUs than ranks)
                backend = os.environ.get("XA_DIST_BACKEND") or (
                    "nccl" if torch.cuda.is_available() else "gloo")
            if backend == "nccl":
                torch.cuda.set_device(local)
            dist.init_process_group(backend=backend, rank=rank, world_size=world)
    return rank, world, local


def view_cost(entry, w: int, h: int) -> float:
    """Relative cost of one grid entry: blur taps over the source plus
    resampling + ORB over the view (view area = w*h*s^2/t)."""
    t, s = float(entry[1]), float(entry[3])
    taps = 0 if t == 1.0 else 2 * max(1, math.ceil(3 * 0.8 * math.sqrt(t * t - 1))) + 1
    return w * h * (taps * 4 + (s * s / t) * (64 + 3.1 * 40))


def lpt_assign(costs: Sequence[float], world: int) -> List[List[int]]:
    """Longest-processing-time-first assignment; deterministic tie-breaks."""
    order = sorted(range(len(costs)), key=lambda i: (-costs[i], i))
    load = [0.0] * world
    out: List[List[int]] = [[] for _ in range(world)]
    for i in order:
        r = min(range(world), key=lambda k: (load[k], k))
        out[r].append(i)
        load[r] += costs[i]
    return [sorted(x) for x in out]


def block_range(n: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous block [lo, hi) of n items for rank (query-block sharding)."""
    base, rem = divmod(n, world)
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)


def _all_gather_np(arr: np.ndarray, world: int, device=None) -> List[np.ndarray]:
    import torch
    import torch.distributed as dist
    t = torch.from_numpy(np.ascontiguousarray(arr))
    if device is not None:
        t = t.to(device)
    n = torch.tensor([t.shape[0]], dtype=torch.int64, device=t.device)
    sizes = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(sizes, n)
    m = int(max(s.item() for s in sizes))
    pad = torch.zeros((m,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
    pad[: t.shape[0]] = t
    bufs = [torch.zeros_like(pad) for _ in range(world)]
    dist.all_gather(bufs, pad)
    return [b[: int(s.item())].cpu().numpy() for b, s in zip(bufs, sizes)]


def argmax_grid_order(counts: Sequence[int]) -> int:
    """pipeline.cpp:142-150: best starts at -1, strict '>' in grid order."""
    best, bi = -1, 0
    for i, c in enumerate(counts):
        if c > best:
            best, bi = int(c), i
    return bi


def coarse_search_sharded(grid: np.ndarray, w: int, h: int, rank: int, world: int,
                          run_entries: Callable[[List[int]], np.ndarray], device=None):
    """run_entries(indices) -> counts for those grid entries on this rank.
    Returns (counts for the whole grid, best index), identical on every rank."""
    grid = np.asarray(grid, np.float64).reshape(-1, 6)
    assign = lpt_assign([view_cost(e, w, h) for e in grid], world)
    mine = assign[rank]
    local = np.asarray(run_entries(mine), np.int32) if mine else np.zeros(0, np.int32)
    payload = np.stack([np.asarray(mine, np.int32), local], 1) if mine else np.zeros((0, 2), np.int32)
    if world > 1:
        parts = _all_gather_np(payload, world, device)
    else:
        parts = [payload]
    counts = np.zeros(len(grid), np.int32)
    for p in parts:
        counts[p[:, 0]] = p[:, 1]
    return counts, argmax_grid_order(counts)


def match_sharded(na: int, rank: int, world: int,
                  run_block: Callable[[int, int], np.ndarray], device=None) -> np.ndarray:
    """run_block(lo, hi) -> (hi-lo, 3) int32 [best_idx, best, second] for queries
    [lo, hi); returns the full (na, 3) table on every rank."""
    lo, hi = block_range(na, world, rank)
    part = np.asarray(run_block(lo, hi), np.int32).reshape(-1, 3)
    if world == 1:
        return part
    return np.concatenate(_all_gather_np(part, world, device), 0)


def pairs_for_rank(n_pairs: int, rank: int, world: int) -> List[int]:
    """Round-robin pair sharding (BASELINE config 5)."""
    return list(range(rank, n_pairs, world))


def coarse_search_pairs_sharded(n_pairs: int, n_entries: int, rank: int, world: int,
                                run_block: Callable[[int, int], np.ndarray], device=None):
    """BASELINE config 5 over `world` ranks: run_block(lo, hi) -> (hi-lo, n_entries)
    int32 per-entry counts for pairs [lo, hi) on this rank's GPU. Returns
    (counts (n_pairs, n_entries), best entry per pair), identical on every rank
    and for every world size (the blocks are gathered in pair order)."""
    lo, hi = block_range(n_pairs, world, rank)
    part = np.asarray(run_block(lo, hi), np.int32).reshape(hi - lo, n_entries) if hi > lo \
        else np.zeros((0, n_entries), np.int32)
    counts = part if world == 1 else np.concatenate(_all_gather_np(part, world, device), 0)
    return counts, [argmax_grid_order(r) for r in counts]
