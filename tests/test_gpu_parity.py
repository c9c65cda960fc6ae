"""GPU parity: the CUDA path through the C-ABI against the CPU oracle and the
reference's own golden vectors.  Integer counts: bit-exact, zero tolerance.

Mirrors the reference's tests: test_star_engine.cpp, test_triangle_engine.cpp,
test_executor.cpp, test_oracle.cpp, test_indexes.cpp (file:line cited inline).
"""
import numpy as np
import pytest

from conftest import load_golden, toy_arrays

pytestmark = pytest.mark.gpu

O_, IN_ = 0, 1


def ctx_of(tm, g):
    return tm.GraphContext.build(g)


def oracle_graph(oracle, g):
    return oracle.build_graph(g.node_count(), g.src, g.dst, g.t)


# --- toy graph (Fig. 1) ---------------------------------------------------------
def test_toy_frozen_census(cuda, tm):
    """test_oracle.cpp 'toy census at delta 10 matches the frozen vector'."""
    frozen = load_golden("toy_frozen.json")["census"]
    g = toy_arrays()
    census = tm.run_parallel(ctx_of(tm, g), tm.RunConfig(delta=10))
    for sig, c in frozen.items():
        assert census.count(sig) == c, sig
    assert census.total() == sum(frozen.values())


def test_toy_reference_counters_all_deltas(cuda, tm):
    ref = load_golden("toy_reference.json")
    g = toy_arrays()
    assert list(g.node_ids) == ref["node_ids"]
    ctx = ctx_of(tm, g)
    for case in ref["cases"]:
        d = case["delta"]
        sp = tm.count_star_pair(ctx, d)
        assert sp.star.cells.tolist() == case["star"], d
        assert sp.pair.cells.tolist() == case["pair"], d
        assert tm.count_triangles(ctx, d).cells.tolist() == case["tri_countall"], d
        assert tm.count_triangles(ctx, d, tm.TriangleMode.removal).cells.tolist() == case["tri_removal"], d
        assert tm.run_parallel(ctx, tm.RunConfig(delta=d)).counts.tolist() == case["census"], d
        assert case["census"] == case["oracle_census"]
        nodes = [pc["node"] for pc in case["per_center"]]
        stars = tm.count_star_pair_items(ctx, d, nodes, [tm.full_star_range(pc["degree"]) for pc in case["per_center"]])
        tris = tm.count_triangles_items(ctx, d, nodes, [tm.full_triangle_range(pc["degree"]) for pc in case["per_center"]])
        for pc, s, t in zip(case["per_center"], stars, tris):
            assert s.star.cells.tolist() == pc["star"], (d, pc["node"])
            assert s.pair.cells.tolist() == pc["pair"], (d, pc["node"])
            assert t.cells.tolist() == pc["tri"], (d, pc["node"])


def test_toy_center_a_worked_increments(cuda, tm):
    """test_star_engine.cpp:16-34: Star[III,o,o,in], Star[III,o,o,o],
    Star[II,o,in,o], Star[II,o,o,o] each 1, nothing else."""
    g = toy_arrays()
    ctx = ctx_of(tm, g)
    a = g.find_node("a")
    r = tm.count_star_pair_at_center(ctx, a, 10, tm.full_star_range(ctx.degree(a)))
    T = tm.StarType
    assert r.star.at(T.isolated_third, O_, O_, IN_) == 1
    assert r.star.at(T.isolated_third, O_, O_, O_) == 1
    assert r.star.at(T.isolated_second, O_, IN_, O_) == 1
    assert r.star.at(T.isolated_second, O_, O_, O_) == 1
    assert int(r.star.cells.sum()) == 4
    assert int(r.pair.cells.sum()) == 0


def test_toy_center_e_triangles(cuda, tm):
    """test_triangle_engine.cpp:19-32."""
    g = toy_arrays()
    ctx = ctx_of(tm, g)
    e = g.find_node("e")
    r = tm.count_triangles_at_center(ctx, e, 10, tm.full_triangle_range(ctx.degree(e)))
    T = tm.TriangleType
    assert r.at(T.closing_last, O_, O_, O_) == 1
    assert r.at(T.closing_middle, O_, IN_, IN_) == 1
    assert int(r.cells.sum()) == 2


def test_toy_sequences_and_pair_index(cuda, tm):
    """test_indexes.cpp:24-75 and 77-99 (device-built S and G)."""
    g = toy_arrays()
    ctx = ctx_of(tm, g)
    n = lambda x: g.find_node(x)
    sa = ctx.sequence(n("a"))
    assert [(r.t, r.other, int(r.dir)) for r in sa] == [
        (4, n("c"), 0), (8, n("c"), 0), (9, n("d"), 1), (11, n("b"), 0), (15, n("c"), 0)]
    se = ctx.sequence(n("e"))
    assert [(r.t, r.other, int(r.dir)) for r in se] == [
        (1, n("d"), 0), (6, n("c"), 0), (14, n("d"), 1), (18, n("d"), 0), (21, n("d"), 1)]
    rel_c = ctx.edges_in_window(n("c"), n("d"), -2 ** 63, 2 ** 63 - 1)
    assert [(t, int(d)) for t, _, d in rel_c] == [(10, 1), (17, 0)]
    rel_d = ctx.edges_in_window(n("d"), n("c"), 4, 14)
    assert [(t, int(d)) for t, _, d in rel_d] == [(10, 0)]
    assert ctx.edges_in_window(n("c"), n("d"), 11, 16) == []
    assert ctx.edges_in_window(n("b"), n("e"), 0, 100) == []


# --- reference golden sweep ------------------------------------------------------
@pytest.fixture(scope="module")
def random_golden():
    return load_golden("random_reference.json")


def test_random_sweep_matches_reference(cuda, tm, random_golden):
    """SPEC acceptance 1/3/4: 48 seeded graphs x 5 deltas, counters + census."""
    for case in random_golden["cases"]:
        g = tm.generate_random_graph(case["nodes"], case["edges"], case["t_max"], case["seed"])
        ctx = ctx_of(tm, g)
        assert tm.auto_degree_threshold(ctx) == case["auto_threshold"]
        for dc in case["deltas"]:
            d = dc["delta"]
            sp = tm.count_star_pair(ctx, d)
            assert sp.star.cells.tolist() == dc["star"], (case["seed"], d)
            assert sp.pair.cells.tolist() == dc["pair"], (case["seed"], d)
            assert tm.count_triangles(ctx, d).cells.tolist() == dc["tri_countall"], (case["seed"], d)
            assert tm.count_triangles(ctx, d, tm.TriangleMode.removal).cells.tolist() == dc["tri_removal"]
            assert tm.run_parallel(ctx, tm.RunConfig(delta=d)).counts.tolist() == dc["census"]
            rem = tm.run_parallel(ctx, tm.RunConfig(delta=d, triangle_mode=tm.TriangleMode.removal))
            assert rem.counts.tolist() == dc["census_removal"]
        ctx.close()


def test_per_center_items_and_range_additivity(cuda, tm, oracle):
    """test_star_engine.cpp:77-121, test_triangle_engine.cpp:63-79 / 130-146."""
    rng = np.random.default_rng(5)
    for seed in (1, 2, 3, 4, 5, 6):
        g = tm.generate_random_graph(12, 150, 40 if seed % 2 else 4000, seed)
        og = oracle_graph(oracle, g)
        ctx = ctx_of(tm, g)
        degs = ctx.degrees()
        for delta in (0, 3, 50, 5000):
            nodes = list(range(g.node_count()))
            stars = tm.count_star_pair_items(ctx, delta, nodes, [tm.full_star_range(int(degs[u])) for u in nodes])
            tris = tm.count_triangles_items(ctx, delta, nodes, [tm.full_triangle_range(int(degs[u])) for u in nodes])
            for u in nodes:
                s = int(degs[u])
                st, pr = oracle.star_pair_at_center(og, u, delta, 0, max(s - 2, 0))
                assert (stars[u].star.cells == st).all() and (stars[u].pair.cells == pr).all()
                assert (tris[u].cells == oracle.triangles_at_center(og, u, delta, 0, max(s - 1, 0))).all()
                # random split points and arbitrary sub-ranges
                for _ in range(3):
                    lo = int(rng.integers(0, s + 1)); hi = int(rng.integers(lo, s + 2))
                    a = tm.count_star_pair_at_center(ctx, u, delta, (lo, hi))
                    st, pr = oracle.star_pair_at_center(og, u, delta, lo, hi)
                    assert (a.star.cells == st).all() and (a.pair.cells == pr).all(), (seed, u, lo, hi)
                    tt = tm.count_triangles_at_center(ctx, u, delta, (lo, hi))
                    assert (tt.cells == oracle.triangles_at_center(og, u, delta, lo, hi)).all()
        oracle.free(og)


def test_live_mask_items(cuda, tm, oracle):
    """Removal-mode center calls with a live mask (triangle_engine.cpp:75-83)."""
    for seed in (3, 9, 27):
        g = tm.generate_random_graph(11, 160, 25 if seed % 2 else 3000, seed)
        og = oracle_graph(oracle, g)
        ctx = ctx_of(tm, g)
        degs = ctx.degrees()
        live = np.ones(11, np.uint8)
        for u in range(11):
            got = tm.count_triangles_at_center(ctx, u, 300, tm.full_triangle_range(int(degs[u])), live)
            exp = oracle.triangles_at_center(og, u, 300, 0, max(int(degs[u]) - 1, 0), live)
            assert (got.cells == exp).all()
            live[u] = 0
        oracle.free(og)


# --- edge cases ----------------------------------------------------------------------
def test_empty_and_tiny_graphs(cuda, tm):
    g = tm.TemporalGraph([], np.zeros(0, np.uint32), np.zeros(0, np.uint32), np.zeros(0, np.int64))
    ctx = ctx_of(tm, g)
    assert tm.run_parallel(ctx, tm.RunConfig(delta=100)).total() == 0
    g = tm.TemporalGraph(["a", "b", "c"], np.zeros(0, np.uint32), np.zeros(0, np.uint32), np.zeros(0, np.int64))
    assert tm.run_parallel(ctx_of(tm, g), tm.RunConfig(delta=5)).total() == 0
    # three parallel edges: one pair instance seen from both ends (test_star_engine.cpp:64-75)
    g = tm.parse_edge_list("a b 1\na b 2\na b 3\n")
    ctx = ctx_of(tm, g)
    r = tm.count_star_pair(ctx, 10)
    assert r.pair.at(O_, O_, O_) == 1 and r.pair.at(IN_, IN_, IN_) == 1
    assert int(r.pair.cells.sum()) == 2 and int(r.star.cells.sum()) == 0
    assert tm.run_parallel(ctx, tm.RunConfig(delta=5)).count("12|12|12") == 1
    # a single triangle lands once in each cell of its class (test_triangle_engine.cpp:82-101)
    g = tm.parse_edge_list("a c 8\nd a 9\nc d 17\n")
    r = tm.count_triangles(ctx_of(tm, g), 9)
    T = tm.TriangleType
    assert r.at(T.closing_last, O_, IN_, O_) == 1
    assert r.at(T.closing_middle, IN_, O_, IN_) == 1
    assert r.at(T.closing_first, O_, IN_, O_) == 1
    assert int(r.cells.sum()) == 3


def test_ties_and_zero_delta(cuda, tm, oracle):
    """test_oracle.cpp:58-71: tied timestamps fit a zero window."""
    g = tm.parse_edge_list("a b 7\na b 7\nb a 7\n")
    assert tm.run_parallel(ctx_of(tm, g), tm.RunConfig(delta=0)).count("12|12|21") == 1
    for seed in range(10):
        g = tm.generate_random_graph(8, 300, 3, seed)  # massive ties
        og = oracle_graph(oracle, g)
        ctx = ctx_of(tm, g)
        for d in (0, 1, 2):
            for rem in (False, True):
                mode = tm.TriangleMode.removal if rem else tm.TriangleMode.count_all
                got = tm.run_parallel(ctx, tm.RunConfig(delta=d, triangle_mode=mode)).counts
                assert (got == oracle.census(og, d, rem)).all(), (seed, d, rem)
        oracle.free(og)


def test_extreme_timestamps_saturate(cuda, tm, oracle):
    """sat_add / sat_sub window bounds (types.hpp:72-89) near int64 limits."""
    big = 2 ** 63 - 1
    for base in (big - 50, -(2 ** 63) + 3):
        rng = np.random.default_rng(abs(base) % 1000)
        n, m = 6, 120
        src = rng.integers(0, n, m).astype(np.uint32)
        dst = ((src + rng.integers(1, n, m)) % n).astype(np.uint32)
        off = rng.integers(0, 40, m)
        t = (np.int64(base) - off.astype(np.int64)) if base > 0 else (np.int64(base) + off.astype(np.int64))
        g = tm.TemporalGraph([str(i) for i in range(n)], src, dst, t)
        og = oracle_graph(oracle, g)
        ctx = ctx_of(tm, g)
        for d in (0, 7, 2 ** 62, big):
            assert (tm.run_parallel(ctx, tm.RunConfig(delta=d)).counts == oracle.census(og, d)).all(), d
        oracle.free(og)


def test_time_span_at_the_narrow_record_boundary(cuda, tm, oracle):
    """u32 time offsets are used while the span is <= 0xFFFFFFFE (searches
    compare offsets against a u32 threshold, 0xFFFFFFFF = every record); a
    span one past that switches to int64 times.  Both sides of the boundary,
    with records clustered at both ends of the span and deltas that reach
    across it."""
    for span in (0xFFFFFFFE, 0xFFFFFFFF, 2 ** 32, 2 ** 32 + 5):
        for base in (0, -(2 ** 40), 2 ** 62):
            rng = np.random.default_rng(span % 977 + abs(base) % 13)
            n, m = 7, 160
            src = rng.integers(0, n, m).astype(np.uint32)
            dst = ((src + rng.integers(1, n, m)) % n).astype(np.uint32)
            off = np.where(rng.random(m) < 0.5, rng.integers(0, 30, m), span - rng.integers(0, 30, m))
            off[0], off[1] = 0, span
            t = np.sort(np.int64(base) + off.astype(np.int64))
            g = tm.TemporalGraph([str(i) for i in range(n)], src, dst, t)
            og = oracle_graph(oracle, g)
            ctx = ctx_of(tm, g)
            for d in (0, 9, 2 ** 31, span - 1, span, 2 ** 33, 2 ** 63 - 1):
                assert (tm.run_parallel(ctx, tm.RunConfig(delta=d)).counts == oracle.census(og, d)).all(), (span, base, d)
            oracle.free(og)


def test_errors_mirror_reference(cuda, tm):
    g = toy_arrays()
    ctx = ctx_of(tm, g)
    with pytest.raises(tm.ConfigError):
        tm.run_parallel(ctx, tm.RunConfig(delta=10, workers=4, triangle_mode=tm.TriangleMode.removal))
    with pytest.raises(tm.ConfigError):
        tm.run_parallel(ctx, tm.RunConfig(delta=-1))
    assert tm.run_parallel(ctx, tm.RunConfig(delta=10, workers=64)).total() > 0
    with pytest.raises(ValueError):
        tm.GraphContext.build(tm.TemporalGraph.from_arrays(3, [0, 1], [1, 5], [1, 2]))


def test_motif_filter(cuda, tm):
    """test_executor.cpp:181-214."""
    g = tm.generate_random_graph(25, 300, 150, 19)
    ctx = ctx_of(tm, g)
    full = tm.run_parallel(ctx, tm.RunConfig(delta=40))
    parts = {}
    for name, f in (("star", tm.MotifFilter(True, False, False)), ("pair", tm.MotifFilter(False, True, False)),
                    ("triangle", tm.MotifFilter(False, False, True))):
        parts[name] = tm.run_parallel(ctx, tm.RunConfig(delta=40, motifs=f))
    for s in tm.all_signatures():
        cat = tm.signature_category(s)
        for name, c in parts.items():
            assert c.count(s) == (full.count(s) if name == cat else 0)


def test_center_partition_sums_to_full(cuda, tm):
    """Multi-GPU data path on one device: partial counters over a degree-cost
    partition sum to the full run (the all-reduce is a plain u64 sum)."""
    g = tm.generate_random_graph(300, 20000, 5000, 11)
    ctx = ctx_of(tm, g)
    for mode in (tm.TriangleMode.count_all, tm.TriangleMode.removal):
        cfg = tm.RunConfig(delta=200, triangle_mode=mode)
        full_raw, full_census = tm.run_parallel_raw(ctx, cfg)
        for world in (2, 3, 8):
            acc = np.zeros(56, np.uint64)
            bounds = [ctx.partition(world, r) for r in range(world)]
            assert bounds[0][0] == 0 and bounds[-1][1] == g.node_count()
            for (b, e), (b2, _) in zip(bounds, bounds[1:]):
                assert e == b2
            for b, e in bounds:
                if b == e:
                    continue
                raw, _ = tm.run_parallel_raw(ctx, cfg, b, e)
                acc += raw.as_array()
            assert (acc == full_raw.as_array()).all()
        merged = tm.merge_census(full_raw.star, full_raw.pair, full_raw.tri, mode)
        assert (merged.counts == full_census).all()


# --- full-size configs --------------------------------------------------------------
def test_config0_uniform_full_size_matches_reference(cuda, tm):
    ref = load_golden("uniform_reference.json")
    from paper_2204_09236_b200 import synth
    n, s, d, t = synth.uniform(ref["nodes"], ref["edges"], ref["t_max"], ref["seed"])
    ctx = tm.GraphContext.build(tm.TemporalGraph.from_arrays(n, s, d, t))
    raw, census = tm.run_parallel_raw(ctx, tm.RunConfig(delta=ref["delta"]))
    assert raw.star.cells.tolist() == ref["star"]
    assert raw.pair.cells.tolist() == ref["pair"]
    assert raw.tri.cells.tolist() == ref["tri_countall"]
    assert census.tolist() == ref["census"]
    assert tm.count_triangles(ctx, ref["delta"], tm.TriangleMode.removal).cells.tolist() == ref["tri_removal"]


def _class_checks(tm, raw, ctx=None, delta=None):
    """Pair complementary-cell equality (SPEC acceptance 3), and -- with a
    graph -- the triangle class sums of the count_all cells equal 3x those of
    the removal cells: the two come from different orientations (degree class
    vs node index) and different forward sequences, so this can fail, unlike
    equality inside a count_all class (the host expands class sums into the
    cells, so that holds by construction)."""
    p = raw.pair.cells
    for c in range(8):
        assert p[c] == p[7 - c]
    if ctx is None:
        return
    rem = tm.count_triangles(ctx, delta, tm.TriangleMode.removal).cells
    all_, once = {}, {}
    for c in range(24):
        sig = tm.tri_cell_signature(c >> 3, (c >> 2) & 1, (c >> 1) & 1, c & 1)
        all_[sig] = all_.get(sig, 0) + int(raw.tri.cells[c])
        once[sig] = once.get(sig, 0) + int(rem[c])
    assert len(all_) == 8
    for sig in all_:
        assert all_[sig] == 3 * once[sig], sig
    assert sum(once.values()) > 0


def test_config1_powerlaw_full_size_properties(cuda, tm):
    """BASELINE config 1 at full size (1M nodes, 10M edges, delta 3600):
    size-independent properties + the reference's census when the golden
    vector was generated (tests/golden/powerlaw_reference.json)."""
    import os
    from paper_2204_09236_b200 import synth
    n, s, d, t = synth.power_law()
    ctx = tm.GraphContext.build(tm.TemporalGraph.from_arrays(n, s, d, t))
    raw, census = tm.run_parallel_raw(ctx, tm.RunConfig(delta=3600))
    _class_checks(tm, raw, ctx, 3600)
    rem = tm.run_parallel(ctx, tm.RunConfig(delta=3600, triangle_mode=tm.TriangleMode.removal))
    assert (rem.counts == census).all()  # mode equivalence (SPEC acceptance 4)
    small = tm.run_parallel(ctx, tm.RunConfig(delta=600))
    assert (small.counts <= census).all()  # delta monotonicity (SPEC acceptance 6)
    path = os.path.join(os.path.dirname(__file__), "golden", "powerlaw_reference.json")
    if os.path.exists(path):
        ref = load_golden("powerlaw_reference.json")
        assert census.tolist() == ref["census"]
    # the BASELINE delta sweep on the same input, vs the reference's census
    path = os.path.join(os.path.dirname(__file__), "golden", "powerlaw_deltas_reference.json")
    if os.path.exists(path):
        ref = load_golden("powerlaw_deltas_reference.json")
        for case in ref["cases"]:
            got = tm.run_parallel(ctx, tm.RunConfig(delta=case["delta"]))
            assert got.counts.tolist() == case["census"], case["delta"]


def test_config2_hubstress_full_size_vs_reference(cuda, tm):
    """BASELINE config 2 at full size (100k nodes, 50M edges with 20 hubs on
    30 % of the edges, bursty unsorted timestamps -> the GPU time sort runs):
    census == the reference's own run_parallel census on the identical input
    (tests/golden/hubstress_reference.json, made by make_golden.py --hubstress),
    for the whole graph and for a 2-way time-slice split summed."""
    import hashlib
    import os
    from paper_2204_09236_b200 import synth
    from paper_2204_09236_b200.distributed import time_slice_bounds, time_slice_mask
    path = os.path.join(os.path.dirname(__file__), "golden", "hubstress_reference.json")
    if not os.path.exists(path):
        pytest.skip("hubstress golden not generated")
    ref = load_golden("hubstress_reference.json")
    n, s, d, t = synth.hub_stress()
    h = hashlib.sha256()
    for a in (s, d, t):
        h.update(np.ascontiguousarray(a).tobytes())
    assert h.hexdigest()[:16] == ref["hash"]  # same input as the reference saw
    delta = ref["delta"]
    census = tm.run_parallel(tm.GraphContext.build(tm.TemporalGraph.from_arrays(n, s, d, t)),
                             tm.RunConfig(delta=delta))
    assert census.counts.tolist() == ref["census"]
    total = np.zeros(56, np.uint64)
    for lo, hi in time_slice_bounds(t, 2):
        keep = time_slice_mask(t, lo, hi, delta)
        raw = tm.count_edges_time_slice(n, s[keep], d[keep], t[keep], tm.RunConfig(delta=delta), lo, hi)
        total += raw.as_array()
    rc = tm.RawCounters.from_array(total)
    merged = tm.merge_census(rc.star, rc.pair, rc.tri, tm.TriangleMode.count_all)
    assert merged.counts.tolist() == ref["census"]


def test_cpp_host_mirror_driver(cuda, tm, oracle):
    """The C++ header mirror (include/tmotif_b200.hpp) used as a reference
    caller would: toy census == frozen vector; random graph == oracle."""
    import os
    import subprocess
    exe = os.path.join(os.path.dirname(__file__), "cpp", "capi_parity")
    out = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stdout + out.stderr
    got = dict((l.split()[0], int(l.split()[1])) for l in out.stdout.splitlines())
    assert got == load_golden("toy_frozen.json")["census"]
    n, m, delta = 80, 4000, 300
    s, d, t = oracle.generate_random_graph(n, m, 20000, 31337)
    inp = "".join(f"{a} {b} {c}\n" for a, b, c in zip(s, d, t))
    out = subprocess.run([exe, str(n), str(delta)], input=inp, capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stdout + out.stderr
    counts = [int(l.split()[1]) for l in out.stdout.splitlines()]
    og = oracle.build_graph(n, s, d, t)
    assert counts == oracle.census(og, delta).tolist()
    # the same graph as an edge-list file read by the GPU reader through the
    # mirror's parse_edge_list / GraphContext(EdgeList) (ids renamed; comment,
    # blank and self-loop lines mixed in)
    import tempfile
    lines = ["# header", ""] + [f"n{a} n{b} {c}" for a, b, c in zip(s, d, t)] + ["n1 n1 5", "# end"]
    with tempfile.NamedTemporaryFile("w", suffix=".txt", delete=False) as f:
        f.write("\r\n".join(lines))
        path = f.name
    out = subprocess.run([exe, "parse", str(delta), path], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stdout + out.stderr
    head, *rest = out.stdout.splitlines()
    assert head.split()[:6] == ["NODES", str(len(set(s) | set(d))), "EDGES", str(m), "DROPPED", "1"]
    assert head.split()[7] == f"n{s[0]}"
    assert [int(l.split()[1]) for l in rest] == oracle.census(og, delta).tolist()
    with open(path, "a") as f:
        f.write("\nn1 n2 notatime\n")
    out = subprocess.run([exe, "parse", str(delta), path], capture_output=True, text=True, timeout=120)
    assert out.returncode == 5 and out.stdout.startswith(f"PARSE_ERROR {len(lines) + 1} line {len(lines) + 1}: "
                                                           "malformed timestamp 'notatime'"), out.stdout
    os.unlink(path)


def test_time_slices_partition_the_census(cuda, tm, oracle):
    """Time-slice partition (multi-GPU without a replicated build): summing the
    slices' raw counters reproduces the whole graph exactly, for slices cut by
    the library (tm_count_edges_time_slice) and for pre-sliced arrays counted
    with first_edge_t_end."""
    from paper_2204_09236_b200.distributed import time_slice_bounds, time_slice_mask
    cases = [tm.generate_random_graph(40, 3000, 400, 5),       # heavy ties
             tm.generate_random_graph(200, 20000, 100000, 9)]
    for g in cases:
        n = g.node_count()
        for delta in (0, 7, 300):
            for mode in (tm.TriangleMode.count_all, tm.TriangleMode.removal):
                cfg = tm.RunConfig(delta=delta, triangle_mode=mode)
                full, census = tm.run_parallel_raw(tm.GraphContext.build(g), cfg)
                for world in (2, 3, 5):
                    acc_lib = np.zeros(56, np.uint64)
                    acc_pre = np.zeros(56, np.uint64)
                    for lo, hi in time_slice_bounds(g.t, world):
                        acc_lib += tm.count_edges_time_slice(n, g.src, g.dst, g.t, cfg, lo, hi).as_array()
                        keep = time_slice_mask(g.t, lo, hi, delta)
                        c2 = tm.RunConfig(delta=delta, triangle_mode=mode, first_edge_t_end=hi)
                        raw = np.zeros(56, np.uint64)
                        tm.count_edges(n, g.src[keep], g.dst[keep], g.t[keep], c2, raw_out=raw)
                        acc_pre += raw
                    assert (acc_lib == full.as_array()).all(), (delta, mode, world)
                    assert (acc_pre == full.as_array()).all(), (delta, mode, world)
                merged = tm.merge_census(full.star, full.pair, full.tri, mode)
                assert (merged.counts == census).all()


def test_repeated_one_shot_counts_graph_replay(cuda, tm, oracle):
    """tm_count_edges called repeatedly with the same buffers runs eagerly once,
    then captures the sync-free half of the step into a CUDA graph and replays
    it.  Every call must equal the oracle, in place data changes must be seen
    by the replay, and both input modes (device pointers, host arrays) and the
    unsorted-input variant must replay correctly."""
    import torch
    n, m, delta = 70, 5000, 200
    s, d, t = oracle.generate_random_graph(n, m, 30000, 99)
    og = oracle.build_graph(n, s, d, t)
    want = oracle.census(og, delta).tolist()
    cfg = tm.RunConfig(delta=delta)
    ds = torch.from_numpy(s.view(np.int32)).cuda()
    dd = torch.from_numpy(d.view(np.int32)).cuda()
    dt = torch.from_numpy(t).cuda()
    st = torch.cuda.Stream()
    for _ in range(4):  # eager, capture + launch, replay, replay
        got = tm.count_edges_device(n, m, ds.data_ptr(), dd.data_ptr(), dt.data_ptr(), cfg, stream=st.cuda_stream)
        assert got.tolist() == want
    # same buffers, new contents (reversed time order -> the unsorted variant)
    rev = np.ascontiguousarray(t[::-1])
    dt.copy_(torch.from_numpy(rev))
    og2 = oracle.build_graph(n, s, d, rev)
    want2 = oracle.census(og2, delta).tolist()
    for _ in range(3):
        got = tm.count_edges_device(n, m, ds.data_ptr(), dd.data_ptr(), dt.data_ptr(), cfg, stream=st.cuda_stream)
        assert got.tolist() == want2
    # same buffers, a shifted time range (the captured time base must follow)
    for shift in (12345, 10 ** 9, 12345):
        sh = np.ascontiguousarray(t + shift)
        dt.copy_(torch.from_numpy(sh))
        og3 = oracle.build_graph(n, s, d, sh)
        want3 = oracle.census(og3, delta).tolist()
        for _ in range(3):
            got = tm.count_edges_device(n, m, ds.data_ptr(), dd.data_ptr(), dt.data_ptr(), cfg,
                                        stream=st.cuda_stream)
            assert got.tolist() == want3
    # a time slice through the replay path (t_end is part of the config); then
    # the same buffers with every time shifted and t_end shifted alike: the
    # count must not change (a stale captured time base would move all times
    # against t_end)
    hi = int(np.sort(t)[m // 2])
    ref = oracle.census_bruteforce_before(og, delta, hi).tolist()
    for shift in (0, 0, 0, 10 ** 6, 10 ** 6, 10 ** 6):
        dt.copy_(torch.from_numpy(np.ascontiguousarray(t + shift)))
        raw = np.zeros(56, np.uint64)
        tm.count_edges_device(n, m, ds.data_ptr(), dd.data_ptr(), dt.data_ptr(),
                              tm.RunConfig(delta=delta, first_edge_t_end=hi + shift), stream=st.cuda_stream,
                              raw_out=raw)
        rc = tm.RawCounters.from_array(raw)
        got = tm.merge_census(rc.star, rc.pair, rc.tri, tm.TriangleMode.count_all)
        assert got.counts.tolist() == ref, shift
    dt.copy_(torch.from_numpy(t))
    # an invalid edge under a replaying entry: rejected (the speculative replay
    # runs on clamped ids and is discarded), then valid data counts again
    bad = s.copy()
    bad[m // 3] = n + 5
    ds.copy_(torch.from_numpy(bad.view(np.int32)))
    with pytest.raises(ValueError):
        tm.count_edges_device(n, m, ds.data_ptr(), dd.data_ptr(), dt.data_ptr(), cfg, stream=st.cuda_stream)
    ds.copy_(torch.from_numpy(s.view(np.int32)))
    for _ in range(2):
        got = tm.count_edges_device(n, m, ds.data_ptr(), dd.data_ptr(), dt.data_ptr(), cfg, stream=st.cuda_stream)
        assert got.tolist() == want
    # motif filters through the replay (the star side stream unused)
    for cfg_m in (tm.RunConfig(delta=delta, motifs=tm.MotifFilter(star=False, pair=False)),
                  tm.RunConfig(delta=delta, motifs=tm.MotifFilter(triangle=False)),
                  tm.RunConfig(delta=delta, triangle_mode=tm.TriangleMode.removal)):
        base = tm.run_parallel(tm.GraphContext.build(tm.TemporalGraph.from_arrays(n, s, d, t)), cfg_m).counts.tolist()
        for _ in range(3):
            got = tm.count_edges_device(n, m, ds.data_ptr(), dd.data_ptr(), dt.data_ptr(), cfg_m,
                                        stream=st.cuda_stream)
            assert got.tolist() == base
    # host arrays (the e2e path)
    hs = torch.from_numpy(s.view(np.int32)).pin_memory()
    hd = torch.from_numpy(d.view(np.int32)).pin_memory()
    ht = torch.from_numpy(t).pin_memory()
    for _ in range(3):
        got = tm.count_edges(n, hs.numpy().view(np.uint32), hd.numpy().view(np.uint32), ht.numpy(), cfg,
                             stream=st.cuda_stream)
        assert got.tolist() == want


def test_async_pipelined_counts(cuda, tm, oracle):
    """tm_count_edges_async / tm_count_edges_wait: batches streamed from pinned
    host memory with two in flight must each equal the oracle's census of the
    batch they were submitted with -- through the staging slots' eager run,
    capture and speculative replay, with data that switches variant (reversed
    time order) or t range under a replaying slot, an invalid batch (reported
    by its wait, neighbours unaffected) and more submissions than slots before
    any wait."""
    import torch
    n, m, delta = 60, 4000, 150
    batches = []
    for seed in range(3):
        s, d, t = oracle.generate_random_graph(n, m, 20000, 300 + seed)
        batches.append((s, d, t))
    s0, d0, t0 = batches[0]
    batches.append((s0, d0, np.ascontiguousarray(t0[::-1])))   # unsorted variant
    batches.append((s0, d0, np.ascontiguousarray(t0 + 10 ** 7)))  # shifted t range
    want = []
    for s, d, t in batches:
        og = oracle.build_graph(n, s, d, t)
        want.append(oracle.census(og, delta).tolist())
        oracle.free(og)
    pinned = [tuple(torch.from_numpy(a.view(np.int32) if a.dtype == np.uint32 else a).pin_memory() for a in b)
              for b in batches]

    def host(i):
        ps, pd, pt = pinned[i]
        return ps.numpy().view(np.uint32), pd.numpy().view(np.uint32), pt.numpy()

    cfg = tm.RunConfig(delta=delta)
    st = torch.cuda.Stream()
    order = [0, 1, 0, 1, 2, 0, 3, 1, 4, 4, 2, 3, 0, 0, 1]
    pend = []
    for i in order:
        pend.append((i, tm.count_edges_async(n, *host(i), cfg, stream=st.cuda_stream)))
        if len(pend) > 1:
            j, p = pend.pop(0)
            assert p.result().tolist() == want[j], j
    for j, p in pend:
        assert p.result().tolist() == want[j], j
    # three submissions before the first wait (the oldest completes internally)
    ps = [(i, tm.count_edges_async(n, *host(i), cfg, stream=st.cuda_stream)) for i in (1, 2, 0)]
    for j, p in reversed(ps):
        assert p.result().tolist() == want[j], j
    # an invalid batch: its wait raises, the next batch is unaffected
    s, d, t = batches[0]
    bad = s.copy()
    bad[m // 2] = n + 3
    pb = torch.from_numpy(bad.view(np.int32)).pin_memory()
    p_bad = tm.count_edges_async(n, pb.numpy().view(np.uint32), host(0)[1], host(0)[2], cfg, stream=st.cuda_stream)
    p_ok = tm.count_edges_async(n, *host(1), cfg, stream=st.cuda_stream)
    with pytest.raises(ValueError):
        p_bad.result()
    assert p_ok.result().tolist() == want[1]
    # a second collection of the same ticket is rejected by the C-ABI
    L = tm.lib()
    assert L.tm_count_edges_wait(p_ok.ticket, None, None) != 0


def test_pair_table_paths_agree(cuda, tm, oracle):
    """The long-window pair table and the P group ends (both built when the
    long windows hold many wedges) against the oracle: the same dense graphs
    counted with each forced on (TM_PAIR_TABLE=1 -> threshold m wedges,
    TM_GROUP_ENDS=1 -> always) and off (=0) in all four combinations,
    including a time slice (first_edge_t_end)."""
    import json
    import subprocess
    import sys
    script = r'''
import json, sys
import numpy as np
sys.path.insert(0, sys.argv[1])
import paper_2204_09236_b200 as tm
out = []
for n, m, tmax, seed, delta in [(30, 4000, 600, 3, 150), (60, 6000, 3000, 8, 400), (12, 2500, 300, 5, 60)]:
    g = tm.generate_random_graph(n, m, tmax, seed)
    raw = np.zeros(56, np.uint64)
    c = tm.count_edges(n, g.src, g.dst, g.t, tm.RunConfig(delta=delta))
    hi = int(np.sort(g.t)[m // 2])
    tm.count_edges(n, g.src, g.dst, g.t, tm.RunConfig(delta=delta, first_edge_t_end=hi), raw_out=raw)
    out.append([c.tolist(), raw.tolist(), hi])
print(json.dumps(out))
'''
    import os
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = {}
    for mode in ("11", "00", "10", "01"):
        env = dict(os.environ, TM_PAIR_TABLE=mode[0], TM_GROUP_ENDS=mode[1])
        r = subprocess.run([sys.executable, "-c", script, root], env=env, capture_output=True, text=True,
                           timeout=300)
        assert r.returncode == 0, r.stderr[-2000:]
        res[mode] = json.loads(r.stdout.strip().splitlines()[-1])
    assert res["11"] == res["00"] == res["10"] == res["01"]
    res["1"] = res["11"]
    for (n, m, tmax, seed, delta), (census, raw, hi) in zip(
            [(30, 4000, 600, 3, 150), (60, 6000, 3000, 8, 400), (12, 2500, 300, 5, 60)], res["1"]):
        s, d, t = oracle.generate_random_graph(n, m, tmax, seed)
        og = oracle.build_graph(n, s, d, t)
        assert census == oracle.census(og, delta).tolist()
        assert sum(raw[32:56]) > 0
        want = oracle.census_bruteforce_before(og, delta, hi).tolist() if m <= 3000 else None
        if want is not None:
            rc = tm.RawCounters.from_array(np.array(raw, np.uint64))
            assert tm.merge_census(rc.star, rc.pair, rc.tri, tm.TriangleMode.count_all).counts.tolist() == want
        oracle.free(og)


# --- boundary semantics (round 2) ---------------------------------------------------
def test_empty_motif_filter_is_all_zero(cuda, tm):
    """executor.cpp:28-29, 161-163, 204-206: an all-false MotifFilter runs no
    pass and merges to the all-zero census (no error)."""
    g = tm.generate_random_graph(25, 300, 150, 19)
    ctx = ctx_of(tm, g)
    assert tm.run_parallel(ctx, tm.RunConfig(delta=40)).total() > 0
    empty = tm.run_parallel(ctx, tm.RunConfig(delta=40, motifs=tm.MotifFilter(False, False, False)))
    assert empty.total() == 0 and not empty.counts.any()
    raw, census = tm.run_parallel_raw(ctx, tm.RunConfig(delta=40, motifs=tm.MotifFilter(False, False, False)))
    assert not raw.as_array().any()
    assert tm.count_edges(g.node_count(), g.src, g.dst, g.t,
                          tm.RunConfig(delta=40, motifs=tm.MotifFilter(False, False, False))).sum() == 0


def test_counter_overflow_detected_exactly_at_2_64(cuda, tm):
    """CounterOverflowError (types.hpp:65-70) exactly when a cell exceeds
    2^64 - 1.  The test hook starts every raw star/pair accumulator cell at
    `bias` on the device, so Pair = bias + count wraps on the GPU at the
    boundary while Star = raw - Pair stays exact: the device wrap counters and
    the host's 128-bit finish must report overflow for bias = 2^64 - max(Pair)
    and not for one less."""
    L = tm.lib()
    g = tm.generate_random_graph(20, 600, 100, 5)
    ctx = ctx_of(tm, g)
    cfg = tm.RunConfig(delta=30)
    raw0, census0 = tm.run_parallel_raw(ctx, cfg)
    pmax = int(raw0.pair.cells.max())
    assert pmax > 0
    try:
        L.tm_debug_acc_bias((1 << 64) - 1 - pmax)  # max cell lands on 2^64 - 1: fine
        raw1, _ = tm.run_parallel_raw(ctx, tm.RunConfig(delta=30, motifs=tm.MotifFilter(True, True, False)))
        assert (raw1.star.cells == raw0.star.cells).all()
        assert int(raw1.pair.cells.max()) == (1 << 64) - 1
        L.tm_debug_acc_bias((1 << 64) - pmax)  # max cell lands on 2^64: overflow
        with pytest.raises(tm.CounterOverflowError):
            tm.run_parallel_raw(ctx, tm.RunConfig(delta=30, motifs=tm.MotifFilter(True, True, False)))
        with pytest.raises(tm.CounterOverflowError):
            tm.count_star_pair(ctx, 30)
        # star-only filter: the pass still runs (executor.cpp:161), so it still throws
        with pytest.raises(tm.CounterOverflowError):
            tm.run_parallel(ctx, tm.RunConfig(delta=30, motifs=tm.MotifFilter(True, False, False)))
        # triangles only: the star pass does not run, nothing overflows
        tri = tm.run_parallel(ctx, tm.RunConfig(delta=30, motifs=tm.MotifFilter(False, False, True)))
        assert tri.total() == sum(int(c) for k, c in enumerate(census0)
                                  if tm.signature_category(tm.all_signatures()[k]) == "triangle")
    finally:
        L.tm_debug_acc_bias(0)
    assert (tm.run_parallel(ctx, cfg).counts == census0).all()


def test_plan_schedule_mirrors_reference(cuda, tm):
    """plan_schedule (executor.cpp:23-52): heavy = degree > thr_d, sharded over
    full_star_range in shard_target steps; every other node light."""
    g = tm.generate_random_graph(40, 2000, 1000, 3)
    ctx = ctx_of(tm, g)
    deg = np.asarray(g.degrees())
    thr = tm.auto_degree_threshold(ctx)
    assert thr == sorted(deg.tolist(), reverse=True)[19]
    plan = tm.plan_schedule(ctx, thr, 7, tm.MotifFilter())
    assert sorted([h.node for h in plan.heavy] + plan.light) == list(range(40))
    for h in plan.heavy:
        assert deg[h.node] > thr
        b, e = tm.full_star_range(int(deg[h.node]))
        assert h.shards[0][0] == b and h.shards[-1][1] == e
        assert all(y - x <= 7 for x, y in h.shards)
        assert all(a[1] == b2[0] for a, b2 in zip(h.shards, h.shards[1:]))
    assert all(deg[u] <= thr for u in plan.light)
    with pytest.raises(tm.ConfigError):
        tm.plan_schedule(ctx, thr, 0, tm.MotifFilter())
    # the plan's items, counted through the per-center API, sum to the full run
    items = [(h.node, r) for h in plan.heavy for r in h.shards] + \
            [(u, tm.full_star_range(int(deg[u]))) for u in plan.light]
    res = tm.count_star_pair_items(ctx, 60, [u for u, _ in items], [r for _, r in items])
    star = sum(r.star.cells.astype(object) for r in res)
    full = tm.count_star_pair(ctx, 60)
    assert [int(x) for x in star] == [int(x) for x in full.star.cells]


def test_time_slice_open_end_keeps_int64_max(cuda, tm, oracle):
    """A last (open) time slice keeps edges with t == INT64_MAX, and a bounded
    slice whose t_hi + delta saturates keeps them too: sliced == unsliced."""
    top = 2 ** 63 - 1
    rng = np.random.default_rng(4)
    n, m = 12, 400
    s = rng.integers(0, n, m).astype(np.uint32)
    d = ((s + 1 + rng.integers(0, n - 1, m)) % n).astype(np.uint32)
    t = (top - rng.integers(0, 60, m)).astype(np.int64)
    t[:40] = top
    for delta in (5, 100, 2 ** 62):
        cfg = tm.RunConfig(delta=delta)
        full = tm.count_edges_time_slice(n, s, d, t, cfg).as_array()
        og = oracle.build_graph(n, s, d, t)
        assert (tm.RawCounters.from_array(full).as_array() ==
                tm.run_parallel_raw(tm.GraphContext.build(tm.TemporalGraph.from_arrays(n, s, d, t)),
                                    cfg)[0].as_array()).all()
        oracle.free(og)
        for cut in (top - 30, top - 1, top):
            acc = tm.count_edges_time_slice(n, s, d, t, cfg, None, cut).as_array() + \
                tm.count_edges_time_slice(n, s, d, t, cfg, cut, None).as_array()
            assert (acc == full).all(), (delta, cut)


def test_async_then_sync_other_key_keeps_pending_entry(cuda, tm, oracle):
    """with both async slots holding speculative replays, a sync
    count on other arrays must not evict (free) the replay entries the pending
    batches still read; every result equals the oracle."""
    import torch
    n, m, delta = 50, 3000, 120
    batches = [oracle.generate_random_graph(n, m, 20000, 900 + k) for k in range(4)]
    want = []
    for s, d, t in batches:
        og = oracle.build_graph(n, s, d, t)
        want.append(oracle.census(og, delta).tolist())
        oracle.free(og)
    pinned = [tuple(torch.from_numpy(a.view(np.int32) if a.dtype == np.uint32 else a).pin_memory() for a in b)
              for b in batches]

    def host(i):
        ps, pd, pt = pinned[i]
        return ps.numpy().view(np.uint32), pd.numpy().view(np.uint32), pt.numpy()

    cfg = tm.RunConfig(delta=delta)
    st = torch.cuda.Stream()
    # warm both slots into speculative replay (eager, capture, replay per slot)
    for k in range(6):
        tm.count_edges_async(n, *host(k % 2), cfg, stream=st.cuda_stream).result()
    p0 = tm.count_edges_async(n, *host(0), cfg, stream=st.cuda_stream)
    p1 = tm.count_edges_async(n, *host(1), cfg, stream=st.cuda_stream)
    for k in (2, 3, 2, 3):  # sync calls with other keys: replay-cache churn
        got = tm.count_edges(n, *batches[k], tm.RunConfig(delta=delta))
        assert got.tolist() == want[k]
    assert p1.result().tolist() == want[1]
    assert p0.result().tolist() == want[0]


def test_error_codes_distinct(cuda, tm):
    """C-ABI codes: ConsistencyError is 10 (the CLI folds it into exit_usage),
    ConfigError 4, CounterOverflowError 3, ParseError 2 (tmotif_main.cpp:20-30)."""
    assert (tm.TM_ERR_PARSE, tm.TM_ERR_OVERFLOW, tm.TM_ERR_CONFIG, tm.TM_ERR_CONSISTENCY) == (2, 3, 4, 10)
    bad_pair = np.zeros(8, np.uint64)
    bad_pair[0] = 1
    with pytest.raises(tm.ConsistencyError):
        tm.merge_census(tm.StarCounter(), tm.PairCounter(bad_pair), tm.TriCounter())


def test_async_eager_batches_overlap_copy(cuda, tm, oracle):
    """Batches counted eagerly by the asynchronous API (replay off: what every
    batch above the replay size takes) run their census when the next batch is
    submitted, behind its host->device copy: each result must still be its own
    batch's census, through waits in order, out of order and a slot reuse."""
    import json
    import os
    import subprocess
    import sys
    script = r'''
import json, sys
import numpy as np
import torch
sys.path.insert(0, sys.argv[1])
import paper_2204_09236_b200 as tm
n, delta = 50, 120
gs = [tm.generate_random_graph(n, 3000, 20000, 40 + k) for k in range(4)]
pin = [tuple(torch.from_numpy(a.view(np.int32) if a.dtype == np.uint32 else a).pin_memory()
             for a in (g.src, g.dst, g.t)) for g in gs]
host = lambda i: (pin[i][0].numpy().view(np.uint32), pin[i][1].numpy().view(np.uint32), pin[i][2].numpy())
cfg = tm.RunConfig(delta=delta)
st = torch.cuda.Stream()
out = []
p = [tm.count_edges_async(n, *host(i), cfg, stream=st.cuda_stream) for i in (0, 1)]
out.append([0, p[0].result().tolist()])
p.append(tm.count_edges_async(n, *host(2), cfg, stream=st.cuda_stream))
out.append([2, p[2].result().tolist()])   # waits out of order: batch 1 still pending
out.append([1, p[1].result().tolist()])
q = [tm.count_edges_async(n, *host(i), cfg, stream=st.cuda_stream) for i in (3, 0, 1)]  # slot reuse before waits
for i, r in zip((3, 0, 1), q):
    out.append([i, r.result().tolist()])
print(json.dumps(out))
'''
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", script, root], env=dict(os.environ, TM_GRAPHS="0"),
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    got = json.loads(r.stdout.strip().splitlines()[-1])
    want = {}
    for k in range(4):
        g = tm.generate_random_graph(50, 3000, 20000, 40 + k)
        og = oracle.build_graph(50, g.src, g.dst, g.t)
        want[k] = oracle.census(og, 120).tolist()
        oracle.free(og)
    assert len(got) == 6
    for i, c in got:
        assert c == want[i], i


def test_async_packed_timestamps(cuda, tm, oracle):
    """Large eager batches send t as per-block i64 bases + offsets packed by
    host threads: u16 offsets per 4096 edges (tm_async_h2d_bytes = 10 B per
    edge) until a batch has a block that does not fit -- that batch takes the
    plain copy of t and later ones pack u32 offsets per 65536 edges (12 B per
    edge).  Sorted input, input unsorted inside blocks (re-based on the block
    minimum), negative and huge timestamps, and a block whose span exceeds 32
    bits (plain copy) must all give the synchronous census of the same arrays."""
    import json
    import os
    import subprocess
    import sys
    script = r"""
import json, sys
import numpy as np
import torch
sys.path.insert(0, sys.argv[1])
import paper_2204_09236_b200 as tm
n, m, delta = 400, 200_000, 50
rng = np.random.default_rng(5)
def graph(kind):
    src = rng.integers(0, n, m).astype(np.uint32)
    dst = (src + 1 + rng.integers(0, n - 1, m).astype(np.uint32)) % n
    t = np.sort(rng.integers(0, 400_000, m)).astype(np.int64)
    if kind == 1:    # unsorted inside blocks (groups of 64 permuted), negative base: u16 from the block minimum
        t = np.concatenate([rng.permutation(g) for g in np.split(t, m // 64)]) - 10**12
    elif kind == 2:  # near the top of int64
        t = t + (2**63 - 1 - 400_000)
    elif kind in (3, 4):  # wholly permuted: blocks span ~400000 (not u16; u32 from the block minimum)
        t = rng.permutation(t) - 10**12
    elif kind == 5:
        t = t + (2**63 - 1 - 400_000)
    elif kind == 6:  # one block spans more than 2^32: plain copy
        t = t.copy(); t[70_000:] += 2**33; t[70_001] -= 2**34
    return src, dst.astype(np.uint32), t
K = 7
out = []
cfg = tm.RunConfig(delta=delta)
st = torch.cuda.Stream()
pins, pend = [], []
for kind in range(K):
    s, d, t = graph(kind)
    p = tuple(torch.from_numpy(a.view(np.int32) if a.dtype == np.uint32 else a).pin_memory() for a in (s, d, t))
    pins.append(p)
    pend.append(tm.count_edges_async(n, p[0].numpy().view(np.uint32), p[1].numpy().view(np.uint32), p[2].numpy(),
                                     cfg, stream=st.cuda_stream))
    sent = tm.async_h2d_bytes()
    out.append(["bytes", kind, sent])
    # kinds 0-2 are in flight together (results one batch late); from kind 3 on
    # each batch is finished before the next is submitted, so the width the
    # pipeline moved to after a fallback is the next batch's
    if kind in (1, 2):
        out.append(["async", kind - 1, pend[kind - 1].result().tolist()])
    if kind >= 3:
        if kind == 3:
            out.append(["async", 2, pend[2].result().tolist()])
        out.append(["async", kind, pend[kind].result().tolist()])
for kind in range(K):
    p = pins[kind]
    out.append(["sync", kind, tm.count_edges(n, p[0].numpy().view(np.uint32), p[1].numpy().view(np.uint32),
                                             p[2].numpy(), cfg, stream=st.cuda_stream).tolist()])
print(json.dumps(out))
"""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", script, root],
                       env=dict(os.environ, TM_GRAPHS="0", TM_H2D_PACK_MIN="1000", TM_HOST_THREADS="4"),
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    got = json.loads(r.stdout.strip().splitlines()[-1])
    res = {(k, i): v for k, i, v in got}
    m = 200_000
    for kind in range(7):
        assert res[("async", kind)] == res[("sync", kind)], kind
        assert sum(res[("sync", kind)]) > 0
    for kind in range(3):  # u16 offsets
        assert res[("bytes", kind)] == m * 10 + 8 * ((m + 4095) // 4096), kind
    # (a fallback's extra plain copy is added when its census is issued)
    assert res[("bytes", 3)] >= m * 10
    for kind in (4, 5):    # u32 offsets from here on
        assert res[("bytes", kind)] == m * 12 + 8 * ((m + 65535) // 65536), kind
    assert res[("bytes", 6)] >= m * 12


def test_unaligned_device_arrays_and_raw_first_pass(cuda, tm, oracle):
    """The node sort's first pass reads 16-byte aligned src / dst / t with TMA
    (RawEdgeLoad); arrays at odd offsets take the packed path.  Both must give
    the oracle's census, at sizes that end inside a sort tile and on tile
    boundaries (1536 edges per tile)."""
    import torch
    n, delta = 300, 200
    for m in (1, 2, 3, 1535, 1536, 1537, 3072, 10_001):
        g = tm.generate_random_graph(n, m, 20_000, 900 + m)
        order = np.argsort(g.t, kind="stable")  # time-ordered input: no re-pack, the raw first pass runs
        src, dst, tt = g.src[order], g.dst[order], g.t[order]
        og = oracle.build_graph(n, src, dst, tt)
        want = oracle.census(og, delta).tolist()
        oracle.free(og)
        for shift in (0, 1, 2, 3):
            pad = np.zeros(shift, np.uint32)
            s = torch.from_numpy(np.concatenate([pad, src]).view(np.int32)).cuda()[shift:]
            d = torch.from_numpy(np.concatenate([pad, dst]).view(np.int32)).cuda()[shift:]
            t = torch.from_numpy(np.concatenate([pad.astype(np.int64), tt])).cuda()[shift:]
            torch.cuda.synchronize()
            got = tm.count_edges_device(n, m, s.data_ptr(), d.data_ptr(), t.data_ptr(), tm.RunConfig(delta=delta))
            assert got.tolist() == want, (m, shift)
