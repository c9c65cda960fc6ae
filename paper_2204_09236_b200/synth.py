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
# GPU (torch) generator for config 2 (same seeded recipe as hub_stress on the
# device, deterministic for a fixed seed on this image's torch/CUDA; the
# reference's golden census uses the numpy twin).
def _torch():
    import torch
    return torch


def _gpu_gen(seed: int):
    torch = _torch()
    g = torch.Generator(device="cuda")
    g.manual_seed(seed)
    return g


def _det_cumsum(x):
    """Deterministic running sum of non-negative float64 values: fixed-point
    (2^-20) integer prefix sum, since a device float scan may associate
    differently from run to run."""
    torch = _torch()
    q = torch.round(x * float(1 << 20)).to(torch.int64)
    return torch.cumsum(q, 0).to(torch.float64) / float(1 << 20)


def _fix_self_loops(src, dst, redraw):
    torch = _torch()
    bad = (src == dst).nonzero().flatten()
    while bad.numel():
        dst[bad] = redraw(bad.numel())
        bad = bad[src[bad] == dst[bad]]
    return dst


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


GPU_CONFIGS = {
    "hubstress_100k_50m": dict(fn=lambda: hub_stress_gpu(), delta=3600),
    # configs 3 and 4 on the counter-based generators below (the golden
    # references were computed by the reference on the identical arrays)
    "triadic_25m_100m": dict(fn=lambda: triadic_hashed(device="cuda"), delta=86_400),
    "powerlaw_50m_600m": dict(fn=lambda: power_law_hashed(device="cuda"), delta=3600, deltas=(600, 3600, 86_400)),
}


# ---------------------------------------------------------------------------
# Counter-based ("hashed") generators for configs 3 and 4.  Every random draw
# is splitmix64 of (seed, stream, index) in wrapping int64 arithmetic, the
# Chung-Lu CDF is an integer prefix sum and the exponential inter-arrivals
# come from an integer fixed-point table, so numpy on the host and torch on
# the device produce bit-identical edge arrays.  That lets the reference run
# on the CPU (tests/golden/make_golden.py) on exactly the input the GPU
# generates at full size (600M edges in HBM in seconds), and a contiguous
# index range of config 4 (time-ordered) is generated on the host without the
# rest of the graph.
_M64 = 1 << 64


def _s64(x: int) -> int:
    x %= _M64
    return x - _M64 if x >= (1 << 63) else x


_C1 = _s64(0xBF58476D1CE4E5B9)
_C2 = _s64(0x94D049BB133111EB)
_GOLD = _s64(0x9E3779B97F4A7C15)


def _mix_int(z: int) -> int:
    z %= _M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) % _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) % _M64
    return _s64(z ^ (z >> 31))


class _NP:
    """numpy backend of the hashed generators."""
    name = "numpy"

    def arange(self, lo, hi):
        return np.arange(lo, hi, dtype=np.int64)

    def const(self, a):
        return np.asarray(a)

    def searchsorted(self, a, v, right):
        return np.searchsorted(a, v, side="right" if right else "left").astype(np.int64)

    def argsort(self, a):
        return np.argsort(a, kind="stable")

    def cumsum(self, a):
        return np.cumsum(a, dtype=np.int64)

    def where(self, c, a, b):
        return np.where(c, a, b)

    def cat(self, xs):
        return np.concatenate(xs)

    def nonzero(self, m):
        return np.nonzero(m)[0]

    def to_out(self, n, src, dst, t):
        return n, src.astype(np.uint32), dst.astype(np.uint32), t.astype(np.int64)


class _TH:
    """torch (cuda) backend of the hashed generators."""
    name = "torch"

    def __init__(self, device="cuda"):
        self.torch = _torch()
        self.device = device

    def arange(self, lo, hi):
        return self.torch.arange(lo, hi, device=self.device, dtype=self.torch.int64)

    def const(self, a):
        return self.torch.from_numpy(np.ascontiguousarray(a)).to(self.device)

    def searchsorted(self, a, v, right):
        return self.torch.searchsorted(a, v, right=right)

    def argsort(self, a):
        return self.torch.argsort(a, stable=True)

    def cumsum(self, a):
        return self.torch.cumsum(a, 0)

    def where(self, c, a, b):
        return self.torch.where(c, a, b)

    def cat(self, xs):
        return self.torch.cat(xs)

    def nonzero(self, m):
        return m.nonzero().flatten()

    def to_out(self, n, src, dst, t):
        return n, src.to(self.torch.int32), dst.to(self.torch.int32), t


def _lsr(x, k):
    return (x >> k) & ((1 << (64 - k)) - 1)


def _mix(z):
    z = (z ^ _lsr(z, 30)) * _C1
    z = (z ^ _lsr(z, 27)) * _C2
    return z ^ _lsr(z, 31)


def _h64(seed, stream, idx):
    """splitmix64 of (seed, stream, index) -> int64 (bit pattern of a u64)."""
    return _mix(idx * _GOLD + _mix_int(seed * 0x10001 + stream * 0x9E37 + 1))


def _uniform_int(seed, stream, idx, bound):
    """Uniform draw in [0, bound) from the hash's top 53 bits (bound < 2^53)."""
    return _lsr(_h64(seed, stream, idx), 11) % bound


_EXP_BITS = 18
_EXP_FRAC = 32
_TAB_CACHE = {}


def _exp_table(mean_gap: float):
    """-ln(u) * mean_gap in 2^-32 fixed point at 2^18 midpoints of u."""
    key = ("exp", mean_gap)
    if key not in _TAB_CACHE:
        u = (np.arange(1 << _EXP_BITS, dtype=np.float64) + 0.5) / float(1 << _EXP_BITS)
        _TAB_CACHE[key] = np.round(-np.log(u) * mean_gap * float(1 << _EXP_FRAC)).astype(np.int64)
    return _TAB_CACHE[key]


def _cl_cdf(n: int, exponent: float):
    """Integer Chung-Lu CDF: weights rank^(-1/exponent) scaled to a 2^52 total."""
    key = ("cl", n, exponent)
    if key not in _TAB_CACHE:
        w = _chung_lu_weights(n, exponent)
        W = np.maximum(np.floor(w * float(1 << 52)), 1.0).astype(np.int64)
        _TAB_CACHE.clear() if len(_TAB_CACHE) > 8 else None
        _TAB_CACHE[key] = np.cumsum(W)
    return _TAB_CACHE[key]


_S_PERM, _S_SRC, _S_DST, _S_GAP = 1, 2, 3, 4


class _HashedPowerLaw:
    """Config 1/4 recipe on the counter-based RNG: Chung-Lu endpoints through a
    random rank->node permutation, self-loops redrawn on further streams,
    timestamps = floor(cumulative exponential inter-arrivals)."""

    def __init__(self, xp, n, mean_gap, seed, exponent):
        self.xp, self.n, self.seed = xp, n, seed
        self.cdf = xp.const(_cl_cdf(n, exponent))
        self.total = int(_cl_cdf(n, exponent)[-1])
        self.tab = xp.const(_exp_table(mean_gap))
        self.perm = xp.argsort(_h64(seed, _S_PERM, xp.arange(0, n)))

    def _node(self, stream, idx):
        x = _uniform_int(self.seed, stream, idx, self.total)
        return self.perm[self.xp.searchsorted(self.cdf, x, True)]

    def endpoints(self, lo, hi):
        xp = self.xp
        idx = xp.arange(lo, hi)
        src = self._node(_S_SRC, idx)
        dst = self._node(_S_DST, idx)
        attempt = 1
        bad = xp.nonzero(src == dst)
        while len(bad):
            dst[bad] = self._node(_S_DST + 16 * attempt, bad + lo)
            bad = bad[src[bad] == dst[bad]]
            attempt += 1
        return src, dst

    def gaps(self, lo, hi):
        h = _h64(self.seed, _S_GAP, self.xp.arange(lo, hi))
        return self.tab[h & ((1 << _EXP_BITS) - 1)]

    def gap_sum(self, lo, chunk=1 << 24):
        s = 0
        for a in range(0, lo, chunk):
            s += int(self.gaps(a, min(lo, a + chunk)).sum())
        return s

    def edges(self, lo, hi, chunk=1 << 26):
        xp = self.xp
        srcs, dsts, ts = [], [], []
        base = self.gap_sum(lo)
        for a in range(lo, hi, chunk):
            b = min(hi, a + chunk)
            s, d = self.endpoints(a, b)
            fx = xp.cumsum(self.gaps(a, b)) + base
            base = int(fx[-1])
            srcs.append(s.to(xp.torch.int32) if xp.name == "torch" else s.astype(np.uint32))
            dsts.append(d.to(xp.torch.int32) if xp.name == "torch" else d.astype(np.uint32))
            ts.append(fx >> _EXP_FRAC)
        return xp.cat(srcs), xp.cat(dsts), xp.cat(ts)


def _backend(device: str):
    """'cpu' = numpy; 'cuda' = torch on the GPU; 'torch-cpu' = torch on the
    host (lets the CPU suite check the torch path against numpy)."""
    if device == "cpu":
        return _NP()
    return _TH("cpu" if device == "torch-cpu" else device)


def power_law_hashed(n: int = 50_000_000, m: int = 600_000_000, mean_gap: float = 0.05, seed: int = 2204,
                     exponent: float = 1.1, lo: int = 0, hi: int | None = None, device: str = "cpu"):
    """Config 4 (and any power-law size) on the counter-based RNG: edges
    [lo, hi) of the m-edge graph, time-ordered, bit-identical on 'cpu' (numpy
    uint32/int64) and 'cuda' (torch int32/int64)."""
    xp = _backend(device)
    hi = m if hi is None else hi
    g = _HashedPowerLaw(xp, n, mean_gap, seed, exponent)
    src, dst, t = g.edges(lo, hi)
    if xp.name == "torch":
        return n, src, dst, t
    return n, src, dst, t.astype(np.int64)


def triadic_hashed(n: int = 25_000_000, m: int = 100_000_000, closure: float = 0.30, delta: int = 86_400,
                   mean_gap: float = 1.0, seed: int = 2204, exponent: float = 1.1, device: str = "cpu"):
    """Config 3 on the counter-based RNG: (1 - closure) power-law edges, then
    closure x m edges each closing an open wedge u->v->w (a random base edge
    u->v and v's first out-edge at or after it) with an edge between u and w
    in a random direction, timestamped uniformly in [0, delta] after the
    wedge's later edge.  Closing edges are appended, so the input is not
    time-ordered (the GPU build's time sort runs)."""
    xp = _backend(device)
    mb = int(m * (1 - closure))
    g = _HashedPowerLaw(xp, n, mean_gap, seed, exponent)
    src, dst, t = g.edges(0, mb)
    if xp.name == "torch":
        src64, dst64 = src.to(xp.torch.int64), dst.to(xp.torch.int64)
    else:
        src64, dst64 = src.astype(np.int64), dst.astype(np.int64)
    span = int(t[-1]) + 1
    key = src64 * span + t
    order = xp.argsort(key)
    s_key, s_t, s_dst = key[order], t[order], dst64[order]
    need = m - mb
    out_s, out_d, out_t = [], [], []
    got, rnd = 0, 0
    while got < need:
        k = int((need - got) * 1.6) + 1024
        idx = xp.arange(0, k)
        e1 = _uniform_int(seed, 100 + 4 * rnd, idx, mb)
        u, v, t1 = src64[e1], dst64[e1], t[e1]
        pos = xp.searchsorted(s_key, v * span + t1, False)
        pos_c = xp.where(pos < mb, pos, pos * 0)
        ok = (pos < mb) & (s_key[pos_c] // span == v)
        w, t2 = s_dst[pos_c], s_t[pos_c]
        ok = ok & (w != u)
        sel = xp.nonzero(ok)
        u, w, t2, sel_idx = u[sel], w[sel], t2[sel], idx[sel]
        flip = (_h64(seed, 101 + 4 * rnd, sel_idx) & 1) == 1
        a = xp.where(flip, w, u)
        b = xp.where(flip, u, w)
        tc = t2 + _uniform_int(seed, 102 + 4 * rnd, sel_idx, delta + 1)
        take = min(len(u), need - got)
        out_s.append(a[:take]); out_d.append(b[:take]); out_t.append(tc[:take])
        got += take
        rnd += 1
    src = xp.cat([src64] + out_s)
    dst = xp.cat([dst64] + out_d)
    t = xp.cat([t] + out_t)
    return xp.to_out(n, src, dst, t)
