"""GPU, BASELINE configs 2-4 at FULL size (50M / 100M / 600M edges).

Bit-exact against the reference's own run_parallel (executor.cpp:149-215,
oracle/_ref, golden values made by tests/golden/make_golden.py on the
counter-based generators synth.triadic_hashed / synth.power_law_hashed, which
produce the identical edge arrays on the host and on the GPU -- pinned here by
the arrays' hash):
  * config 3 (triadic 25M / 100M) whole, delta 3600 and 86400;
  * config 4 (power-law 50M / 600M): 10M-edge contiguous time slices, one at
    the start of the stream and one mid-stream, at delta 600, 3600 and 86400,
    and the whole 600M edges at the deltas config4_full_reference.json holds;
plus size-independent properties of the full 600M-edge result (pair complement
symmetry, count_all census == removal census, delta monotonicity, center
partitions summing to the whole) and bit-exact agreement with the C oracle on
a time slice of each config's input."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _pair_checks(raw):
    p = raw.pair.cells
    for c in range(8):
        assert p[c] == p[7 - c]


def _hash(src, dst, t):
    """tests/golden/make_golden.py edge_hash of device arrays."""
    import hashlib
    h = hashlib.sha256()
    h.update(src.cpu().numpy().view(np.uint32).tobytes())
    h.update(dst.cpu().numpy().view(np.uint32).tobytes())
    h.update(t.cpu().numpy().astype(np.int64).tobytes())
    return h.hexdigest()[:16]


def _census_device(tm, n, src, dst, t, delta):
    import torch
    torch.cuda.synchronize()
    return tm.count_edges_device(n, src.numel(), src.data_ptr(), dst.data_ptr(), t.data_ptr(),
                                 tm.RunConfig(delta=delta))


def _device_ctx(tm, n, src, dst, t):
    import torch
    torch.cuda.synchronize()
    return tm.GraphContext.build_device(n, src.data_ptr(), dst.data_ptr(), t.data_ptr(), src.numel())


def _slice_parity(tm, oracle, n, src, dst, t, delta, edges):
    """Oracle vs GPU on the earliest `edges` edges in time order (ingestion
    order kept), relabelled to a compact node range."""
    import torch
    order = torch.argsort(t, stable=True)[:edges].sort().values
    s = src[order].cpu().numpy().astype(np.int64)
    d = dst[order].cpu().numpy().astype(np.int64)
    tt = t[order].cpu().numpy()
    ids, inv = np.unique(np.concatenate([s, d]), return_inverse=True)
    s2 = inv[:len(s)].astype(np.uint32)
    d2 = inv[len(s):].astype(np.uint32)
    g = tm.TemporalGraph.from_arrays(len(ids), s2, d2, tt)
    ctx = tm.GraphContext.build(g)
    og = oracle.build_graph(len(ids), s2, d2, tt)
    for rem in (False, True):
        mode = tm.TriangleMode.removal if rem else tm.TriangleMode.count_all
        got = tm.run_parallel(ctx, tm.RunConfig(delta=delta, triangle_mode=mode)).counts
        assert (got == oracle.census(og, delta, rem)).all(), rem
    oracle.free(og)


def _full_checks(tm, ctx, delta, smaller_delta=None):
    raw, census = tm.run_parallel_raw(ctx, tm.RunConfig(delta=delta))
    _pair_checks(raw)
    rem = tm.run_parallel(ctx, tm.RunConfig(delta=delta, triangle_mode=tm.TriangleMode.removal))
    assert (rem.counts == census).all()
    acc = np.zeros(56, np.uint64)
    for r in range(4):
        b, e = ctx.partition(4, r)
        if b < e:
            acc += tm.run_parallel_raw(ctx, tm.RunConfig(delta=delta), b, e)[0].as_array()
    assert (acc == raw.as_array()).all()
    if smaller_delta is not None:
        small = tm.run_parallel(ctx, tm.RunConfig(delta=smaller_delta))
        assert (small.counts <= census).all()
    return census


def test_config2_hub_stress(cuda, tm, oracle):
    from paper_2204_09236_b200 import synth
    n, src, dst, t = synth.hub_stress_gpu()
    _slice_parity(tm, oracle, n, src, dst, t, 3600, 60_000)
    ctx = _device_ctx(tm, n, src, dst, t)
    census = _full_checks(tm, ctx, 3600, 600)
    assert int(census.sum()) > 0


def test_config3_triadic_full_size_vs_reference(cuda, tm, oracle):
    """config 3 whole (100M edges, unordered input: the GPU time sort runs)
    against the reference's run_parallel census at delta 3600 and 86400."""
    import torch
    from conftest import load_golden
    from paper_2204_09236_b200 import synth
    ref = load_golden("triadic_reference.json")
    kw = {k: ref[k] for k in ("n", "m", "closure", "delta", "mean_gap", "seed")}
    n, src, dst, t = synth.triadic_hashed(**kw, device="cuda")
    assert src.numel() == ref["edges"]
    assert _hash(src, dst, t) == ref["hash"]
    assert bool((t[1:] < t[:-1]).any())  # exercises the GPU time sort
    for case in ref["cases"]:
        got = _census_device(tm, n, src, dst, t, case["delta"])
        assert got.tolist() == case["census"], case["delta"]
    _slice_parity(tm, oracle, n, src, dst, t, 86_400, 25_000)
    ctx = _device_ctx(tm, n, src, dst, t)
    _full_checks(tm, ctx, 86_400, 3600)


def test_config4_slices_vs_reference_and_full_size(cuda, tm, oracle):
    """config 4 (600M edges generated on the GPU): each golden 10M-edge time
    slice bit-exact against the reference at delta 600 / 3600 / 86400, then
    the full-size properties."""
    import torch
    from conftest import load_golden
    from paper_2204_09236_b200 import synth
    ref = load_golden("config4_slices_reference.json")
    n, src, dst, t = synth.power_law_hashed(ref["n"], ref["m"], ref["mean_gap"], ref["seed"], device="cuda")
    assert bool((t[1:] >= t[:-1]).all())
    for sl in ref["slices"]:
        lo, hi = sl["lo"], sl["hi"]
        s_, d_, t_ = src[lo:hi].contiguous(), dst[lo:hi].contiguous(), t[lo:hi].contiguous()
        assert _hash(s_, d_, t_) == sl["hash"], (lo, hi)
        for case in sl["cases"]:
            got = _census_device(tm, n, s_, d_, t_, case["delta"])
            assert got.tolist() == case["census"], (lo, hi, case["delta"])
        del s_, d_, t_
    _slice_parity(tm, oracle, n, src, dst, t, 600, 100_000)
    # the whole 600M edges against the reference's run_parallel on the same
    # input (config4_full_reference.json, made on the GPU box's host)
    full = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "config4_full_reference.json")
    if os.path.exists(full):
        fref = load_golden("config4_full_reference.json")
        assert fref["edges"] == src.numel()
        assert _hash(src, dst, t) == fref["hash"]
        for case in fref["cases"]:
            got = _census_device(tm, n, src, dst, t, case["delta"])
            assert got.tolist() == case["census"], ("full", case["delta"])
    ctx = _device_ctx(tm, n, src, dst, t)
    prev = None
    for delta in (600, 3600, 86_400):
        raw, census = tm.run_parallel_raw(ctx, tm.RunConfig(delta=delta))
        _pair_checks(raw)
        if prev is not None:
            assert (census >= prev).all()
        prev = census
    _full_checks(tm, ctx, 3600)
