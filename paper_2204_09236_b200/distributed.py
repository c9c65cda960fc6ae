"""Multi-GPU plumbing: one process per GPU, the 56 raw u64 counters combined
by one all-reduce (NCCL over NVLink on GPUs; gloo in the CPU tests), then
merge_census on every rank.  Two exact partitions of the work:

* time slices (default): rank r holds the edges with t in [tau_r,
  tau_{r+1} + delta) and counts the instances whose earliest edge has t in
  [tau_r, tau_{r+1}).  Every instance has exactly one earliest edge, so the
  slices partition the census; each rank builds only its slice's indexes, so
  the index build scales too.
* center ranges (north_star): graph replicated, centers split by a
  degree-cost prefix sum (tm_partition_centers).

This is the GPU analogue of HARE's inter-node split (executor.cpp:23-52 plan,
executor.cpp:96-139 worker pool + reduction).
"""
from __future__ import annotations

from typing import List, Tuple

import numpy as np


def partition_bounds(cost_prefix: np.ndarray, world: int) -> List[Tuple[int, int]]:
    """Split centers [0, n) into `world` contiguous ranges of ~equal cost.

    cost_prefix[u] = sum of cost(x) for x < u (length n + 1), e.g.
    |S| offsets + |F| offsets as tm_partition_centers uses
    (tm_capi.cu).  Boundary r is the first u with prefix >= total*r/world."""
    cp = np.asarray(cost_prefix, np.uint64)
    n = len(cp) - 1
    total = int(cp[-1])
    out = []
    bounds = [0]
    for r in range(1, world):
        target = total * r // world
        bounds.append(int(np.searchsorted(cp, np.uint64(target), side="left")))
    bounds.append(n)
    for r in range(world):
        out.append((min(bounds[r], n), min(bounds[r + 1], n)))
    return out


def allreduce_counters(raw: np.ndarray, group=None, device=None) -> np.ndarray:
    """Sum 56 u64 counters across ranks.  u64 -> i64 reinterpretation keeps the
    sum exact modulo 2^64, which is the counters' own arithmetic."""
    import torch
    import torch.distributed as dist
    a = np.ascontiguousarray(raw, np.uint64).view(np.int64)
    t = torch.from_numpy(a.copy())
    if device is not None:
        t = t.to(device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return t.cpu().numpy().view(np.uint64).copy()


def run_distributed(ctx, config, rank: int, world: int, group=None, device=None):
    """Each rank counts its center range on its GPU; one all-reduce; merge."""
    from . import tmotif as tm
    b, e = ctx.partition(world, rank)
    if b < e:
        raw, _ = tm.run_parallel_raw(ctx, config, b, e)
        arr = raw.as_array()
    else:
        arr = np.zeros(56, np.uint64)
    tot = allreduce_counters(arr, group, device)
    rc = tm.RawCounters.from_array(tot)
    return tm.merge_census(rc.star, rc.pair, rc.tri, config.triangle_mode)


def time_slice_bounds(t, world: int) -> List[Tuple[object, object]]:
    """Per-rank [lo, hi) first-edge time bounds balanced by edge count
    (None = open end).  Deterministic for the same t on every rank."""
    ts = np.asarray(t, np.int64)
    if len(ts) > 1 and not bool(np.all(ts[1:] >= ts[:-1])):
        ts = np.sort(ts)
    m = len(ts)
    cuts = [int(ts[(r * m) // world]) for r in range(1, world)] if m else []
    lows = [None] + cuts
    highs = cuts + [None]
    return list(zip(lows, highs))


def time_slice_mask(t, lo, hi, delta: int) -> np.ndarray:
    """Edges a rank needs: t in [lo, hi + delta) (saturating at the int64 ends)."""
    t = np.asarray(t, np.int64)
    keep = np.ones(len(t), bool)
    if lo is not None:
        keep &= t >= lo
    if hi is not None:
        top = hi + delta if hi <= (2 ** 63 - 1) - delta else None
        if top is not None:
            keep &= t < top
    return keep
