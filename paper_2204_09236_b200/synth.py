"""Seeded synthetic temporal graphs for the BASELINE.json configs.

The reference publishes no datasets for this path; these generators stand in
with the shapes, sizes and value distributions BASELINE.json names.  Output is
ingestion-order (src u32, dst u32, t i64) numpy arrays, self-loops rejected.
"""
from __future__ import annotations

import numpy as np


def _reject_self_loops(rng, src, dst, sampler):
    bad = np.nonzero(src == dst)[0]
    while len(bad):
        dst[bad] = sampler(len(bad))
        bad = bad[src[bad] == dst[bad]]
    return dst


def uniform(n: int = 10_000, m: int = 200_000, t_max: int = 999_999, seed: int = 2204):
    """config 0: uniform multigraph, t uniform in [0, 1e6).  Uses the
    reference's own generator (graph.cpp:140) so the CPU reference can
    regenerate the identical input."""
    from .tmotif import generate_random_graph
    g = generate_random_graph(n, m, t_max, seed)
    return n, g.src, g.dst, g.t


def _chung_lu_weights(n: int, exponent: float = 1.1):
    r = np.arange(1, n + 1, dtype=np.float64)
    w = r ** (-1.0 / exponent)
    return w / w.sum()


def _cdf_sampler(rng, cdf, perm):
    def draw(k):
        x = np.searchsorted(cdf, rng.random(k), side="right")
        np.minimum(x, len(cdf) - 1, out=x)
        return perm[x].astype(np.uint32)
    return draw


def power_law(n: int = 1_000_000, m: int = 10_000_000, mean_gap: float = 1.0, seed: int = 2204,
              exponent: float = 1.1):
    """config 1 / 5: Chung-Lu endpoints, out/in weights ~ rank^(-1/1.1)
    (degree exponent ~2.1), one shared random rank->node permutation;
    timestamps = cumulative exponential inter-arrivals (mean `mean_gap` s),
    floored to int64 seconds."""
    rng = np.random.default_rng(seed)
    cdf = np.cumsum(_chung_lu_weights(n, exponent))
    perm = rng.permutation(n).astype(np.uint32)
    draw = _cdf_sampler(rng, cdf, perm)
    src = draw(m)
    dst = draw(m)
    dst = _reject_self_loops(rng, src, dst, draw)
    t = np.floor(np.cumsum(rng.exponential(mean_gap, m))).astype(np.int64)
    return n, src, dst, t


def hub_stress(n: int = 100_000, m: int = 50_000_000, hubs: int = 20, hub_share: float = 0.30,
               burst: int = 50, burst_span: float = 10.0, burst_gap: float = 600.0, seed: int = 2204):
    """config 2: the top `hubs` nodes are endpoints of `hub_share` of edges,
    other endpoints uniform; Poisson bursts of `burst` edges within
    `burst_span` s, burst starts exponentially spaced (mean `burst_gap` s)."""
    rng = np.random.default_rng(seed)
    p = 1.0 - np.sqrt(1.0 - hub_share)  # per-endpoint hub probability
    hub_ids = rng.choice(n, hubs, replace=False).astype(np.uint32)

    def draw(k):
        out = rng.integers(0, n, k, dtype=np.uint32)
        h = rng.random(k) < p
        out[h] = hub_ids[rng.integers(0, hubs, int(h.sum()))]
        return out

    src = draw(m)
    dst = draw(m)
    dst = _reject_self_loops(rng, src, dst, draw)
    nb = (m + burst - 1) // burst
    starts = np.cumsum(rng.exponential(burst_gap, nb))
    t = np.repeat(starts, burst)[:m] + rng.random(m) * burst_span
    t = np.floor(t).astype(np.int64)
    return n, src, dst, t


CONFIGS = {
    "uniform_10k_200k": dict(fn=uniform, delta=1000),
    "powerlaw_1m_10m": dict(fn=power_law, delta=3600),
    "hubstress_100k_50m": dict(fn=hub_stress, delta=3600),
}
