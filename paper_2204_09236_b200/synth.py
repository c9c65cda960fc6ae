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


# ---------------------------------------------------------------------------
# GPU (torch) generators for the large configs: same seeded recipe on the
# device, deterministic for a fixed seed on this image's torch/CUDA.
def _torch():
    import torch
    return torch


def _gpu_gen(seed: int):
    torch = _torch()
    g = torch.Generator(device="cuda")
    g.manual_seed(seed)
    return g


_CDF_CACHE = {}


def _gpu_cdf(n, exponent):
    """Chung-Lu CDF computed on the host (sequential, bit-reproducible) and
    uploaded once: a device float scan is not run-to-run deterministic."""
    torch = _torch()
    key = (n, exponent)
    if key not in _CDF_CACHE:
        _CDF_CACHE.clear()
        _CDF_CACHE[key] = torch.from_numpy(np.cumsum(_chung_lu_weights(n, exponent))).cuda()
    return _CDF_CACHE[key]


def _det_cumsum(x):
    """Deterministic running sum of non-negative float64 values: fixed-point
    (2^-20) integer prefix sum, since a device float scan may associate
    differently from run to run."""
    torch = _torch()
    q = torch.round(x * float(1 << 20)).to(torch.int64)
    return torch.cumsum(q, 0).to(torch.float64) / float(1 << 20)


def _chung_lu_draw(n, k, exponent, gen, perm):
    torch = _torch()
    cdf = _gpu_cdf(n, exponent)
    u = torch.rand(k, device="cuda", dtype=torch.float64, generator=gen)
    idx = torch.searchsorted(cdf, u, right=True).clamp_(max=n - 1)
    return perm[idx]


def _fix_self_loops(src, dst, redraw):
    torch = _torch()
    bad = (src == dst).nonzero().flatten()
    while bad.numel():
        dst[bad] = redraw(bad.numel())
        bad = bad[src[bad] == dst[bad]]
    return dst


def power_law_gpu(n: int, m: int, mean_gap: float, seed: int = 2204, exponent: float = 1.1):
    """config 4 recipe on the GPU: Chung-Lu (weights ~ rank^(-1/1.1)), shared
    random rank->node permutation, cumulative exponential inter-arrivals."""
    torch = _torch()
    gen = _gpu_gen(seed)
    perm = torch.randperm(n, device="cuda", generator=gen).to(torch.int64)
    draw = lambda k: _chung_lu_draw(n, k, exponent, gen, perm)
    src = draw(m)
    dst = _fix_self_loops(src, draw(m), draw)
    gaps = torch.empty(m, device="cuda", dtype=torch.float64).exponential_(1.0 / mean_gap, generator=gen)
    t = torch.floor(_det_cumsum(gaps)).to(torch.int64)
    return n, src.to(torch.int32), dst.to(torch.int32), t


def hub_stress_gpu(n: int = 100_000, m: int = 50_000_000, hubs: int = 20, hub_share: float = 0.30,
                   burst: int = 50, burst_span: float = 10.0, burst_gap: float = 600.0, seed: int = 2204):
    """config 2 on the GPU (same recipe as hub_stress)."""
    torch = _torch()
    gen = _gpu_gen(seed)
    p = 1.0 - (1.0 - hub_share) ** 0.5
    hub_ids = torch.randperm(n, device="cuda", generator=gen)[:hubs]

    def draw(k):
        out = torch.randint(0, n, (k,), device="cuda", generator=gen)
        h = torch.rand(k, device="cuda", generator=gen) < p
        nh = int(h.sum())
        out[h] = hub_ids[torch.randint(0, hubs, (nh,), device="cuda", generator=gen)]
        return out

    src = draw(m)
    dst = _fix_self_loops(src, draw(m), draw)
    nb = (m + burst - 1) // burst
    starts = _det_cumsum(torch.empty(nb, device="cuda", dtype=torch.float64)
                         .exponential_(1.0 / burst_gap, generator=gen))
    t = starts.repeat_interleave(burst)[:m] + torch.rand(m, device="cuda", dtype=torch.float64,
                                                          generator=gen) * burst_span
    return n, src.to(torch.int32), dst.to(torch.int32), torch.floor(t).to(torch.int64)


def triadic_gpu(n: int = 25_000_000, m: int = 100_000_000, closure: float = 0.30, delta: int = 86_400,
                mean_gap: float = 1.0, seed: int = 2204, exponent: float = 1.1):
    """config 3: (1 - closure) Chung-Lu edges with cumulative exponential
    timestamps; closure share closes an open wedge u->v->w (w's edge taken as
    v's first out-edge at or after the u->v edge) with an edge between u and w
    in a random direction, timestamped uniformly within [0, delta] after the
    wedge's later edge.  The result is NOT time-ordered (closing edges are
    appended), so the GPU build's time sort runs."""
    torch = _torch()
    gen = _gpu_gen(seed)
    mb = int(m * (1 - closure))
    n_, src, dst, t = power_law_gpu(n, mb, mean_gap, seed, exponent)
    src = src.to(torch.int64)
    dst = dst.to(torch.int64)
    # out-adjacency of the base edges by (src, t)
    key = src * (t.max() + 1) + t
    order = torch.argsort(key, stable=True)
    s_src, s_t, s_dst = src[order], t[order], dst[order]
    starts = torch.searchsorted(s_src, torch.arange(n + 1, device="cuda"))
    need = m - mb
    out_s, out_d, out_t = [], [], []
    got = 0
    while got < need:
        k = int((need - got) * 1.6) + 1024
        e1 = torch.randint(0, mb, (k,), device="cuda", generator=gen)
        u, v, t1 = src[e1], dst[e1], t[e1]
        lo, hi = starts[v], starts[v + 1]
        # first out-edge of v at or after t1 (binary search in v's run)
        pos = torch.searchsorted(s_src * (t.max() + 1) + s_t, v * (t.max() + 1) + t1)
        ok = (pos < hi) & (pos >= lo)
        pos = torch.where(ok, pos, torch.zeros_like(pos))
        w, t2 = s_dst[pos], s_t[pos]
        ok &= (w != u)
        u, w, t2 = u[ok], w[ok], t2[ok]
        flip = torch.rand(u.numel(), device="cuda", generator=gen) < 0.5
        a = torch.where(flip, w, u)
        b = torch.where(flip, u, w)
        tc = t2 + torch.randint(0, delta + 1, (u.numel(),), device="cuda", generator=gen)
        take = min(u.numel(), need - got)
        out_s.append(a[:take]); out_d.append(b[:take]); out_t.append(tc[:take])
        got += take
    src = torch.cat([src] + out_s).to(torch.int32)
    dst = torch.cat([dst] + out_d).to(torch.int32)
    t = torch.cat([t] + out_t)
    return n, src, dst, t


GPU_CONFIGS = {
    "hubstress_100k_50m": dict(fn=lambda: hub_stress_gpu(), delta=3600),
    "triadic_25m_100m": dict(fn=lambda: triadic_gpu(), delta=86_400),
    "powerlaw_50m_600m": dict(fn=lambda: power_law_gpu(50_000_000, 600_000_000, 0.05), deltas=(600, 3600, 86_400)),
}
