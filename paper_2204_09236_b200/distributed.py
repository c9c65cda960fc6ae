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
    """Exact cross-rank sum of 56 u64 counters.  Each counter travels as two
    32-bit halves in int64 words (a sum over <= 2^31 ranks cannot wrap), and
    the totals are recombined with Python integers: a total past 2^64 - 1
    raises CounterOverflowError, as the reference's checked merge of worker
    partials does (executor.cpp:173-179, types.hpp:65-70)."""
    import torch
    import torch.distributed as dist
    from .tmotif import CounterOverflowError
    a = np.ascontiguousarray(raw, np.uint64)
    halves = np.empty(2 * len(a), np.int64)
    halves[0::2] = (a & np.uint64(0xFFFFFFFF)).astype(np.int64)
    halves[1::2] = (a >> np.uint64(32)).astype(np.int64)
    t = torch.from_numpy(halves)
    if device is not None:
        t = t.to(device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    h = t.cpu().numpy()
    tot = [int(lo) + (int(hi) << 32) for lo, hi in zip(h[0::2], h[1::2])]
    if any(x >> 64 for x in tot):
        raise CounterOverflowError("motif counter overflow in the cross-rank merge")
    return np.array(tot, dtype=np.uint64)


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


def time_slice_bounds(t, world: int, delta=None) -> List[Tuple[object, object]]:
    """Per-rank [lo, hi) first-edge time bounds (None = open end),
    deterministic for the same t on every rank.  Without `delta` they are
    edge-count quantiles; with it, quantiles of an estimated work
    w_e = 1 + n_delta(e), n_delta(e) = edges with t in [t_e, t_e + delta]: a
    burst's edges have long windows at every center and weigh more, while a
    stationary stream (configs 1 and 4) keeps the edge-count split."""
    ts = np.asarray(t, np.int64)
    if len(ts) > 1 and not bool(np.all(ts[1:] >= ts[:-1])):
        ts = np.sort(ts)
    m = len(ts)
    if not m:
        cuts = []
    elif delta is None:
        cuts = [int(ts[(r * m) // world]) for r in range(1, world)]
    else:
        # work weights on every k-th edge (k = 1 up to 4M edges): the bounds
        # only need the quantiles of the cumulative work, and every bound
        # choice is exact -- a coarse sample only moves the balance
        k = max(1, m // (1 << 22))
        tsam = ts[::k]
        top = tsam + np.minimum(np.int64(delta), np.int64(2 ** 63 - 1) - tsam)
        w = 1 + (np.searchsorted(ts, top, side="right") - np.arange(0, m, k))
        cw = np.cumsum(w, dtype=np.float64)
        cuts = [int(tsam[min(len(tsam) - 1, int(np.searchsorted(cw, cw[-1] * r / world)))]) for r in range(1, world)]
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
