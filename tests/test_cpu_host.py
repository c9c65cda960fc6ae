"""CPU: the C-ABI library loads and exports every declared symbol, and the
host-side logic (taxonomy, merge, generator, parser) matches the reference's
own tests (test_motifs.cpp, test_graph.cpp).  No compute calls need a GPU."""
import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT, has_cuda, load_golden

O_, IN_ = 0, 1


def header_symbols():
    text = open(os.path.join(ROOT, "include", "tmotif_b200.h")).read()
    return sorted(set(re.findall(r"\b(tm_[a-z_0-9]+)\s*\(", text)))


def test_library_exports_every_declared_symbol(tm):
    lib = ctypes.CDLL(tm.tmotif.LIB_PATH)
    syms = header_symbols()
    assert len(syms) >= 25
    for s in syms:
        assert hasattr(lib, s), s


def test_no_device_means_error_not_fallback(tm):
    if has_cuda():
        pytest.skip("device present")
    g = tm.generate_random_graph(10, 50, 100, 1)
    with pytest.raises(tm.DeviceError):
        tm.GraphContext.build(g)
    with pytest.raises(tm.DeviceError):
        tm.count_edges(10, g.src, g.dst, g.t, tm.RunConfig(delta=5))


def test_signatures_and_cell_maps(tm):
    gold = load_golden("random_reference.json")["signatures"]
    assert tm.all_signatures() == gold
    stars = {tm.star_cell_signature(t, a, b, c) for t in range(3) for a in (0, 1) for b in (0, 1) for c in (0, 1)}
    assert len(stars) == 24 and all(tm.signature_category(s) == "star" for s in stars)
    assert tm.star_cell_signature(2, O_, O_, IN_) == "12|12|31"
    assert tm.star_cell_signature(0, IN_, O_, IN_) == "12|23|32"
    fib = {}
    for a in (0, 1):
        for b in (0, 1):
            for c in (0, 1):
                s = tm.pair_cell_signature(a, b, c)
                assert s == tm.pair_cell_signature(1 - a, 1 - b, 1 - c)
                fib[s] = fib.get(s, 0) + 1
    assert len(fib) == 4 and set(fib.values()) == {2}
    assert tm.pair_cell_signature(O_, IN_, O_) == "12|21|12"
    tri = {}
    for t in range(3):
        for a in (0, 1):
            for b in (0, 1):
                for c in (0, 1):
                    tri.setdefault(tm.tri_cell_signature(t, a, b, c), set()).add(t)
    assert len(tri) == 8 and all(v == {0, 1, 2} for v in tri.values())
    m25 = tm.tri_cell_signature(2, O_, IN_, O_)
    assert m25 == tm.tri_cell_signature(1, IN_, O_, IN_) == tm.tri_cell_signature(0, O_, IN_, O_) == "12|31|23"
    assert tm.tri_cell_signature(2, O_, O_, O_) == "12|13|23"


def test_canonical_signature(tm):
    assert tm.canonical_signature([(2, 3), (2, 3), (1, 2)]) == "12|12|31"
    assert tm.canonical_signature([(1, 0), (0, 1), (1, 0)]) == "12|21|12"
    assert tm.canonical_signature([(0, 3), (1, 3), (1, 0)]) == "12|32|31"
    assert tm.canonical_signature([(5, 9), (9, 7), (7, 5)]) == tm.canonical_signature([(100, 2), (2, 55), (55, 100)])
    with pytest.raises(tm.ClassificationError):
        tm.canonical_signature([(0, 1), (2, 3), (0, 1)])
    with pytest.raises(tm.ClassificationError):
        tm.canonical_signature([(0, 0), (0, 1), (0, 1)])


def test_labels(tm):
    for s, l in {"12|12|12": "M_55", "12|12|31": "M_63", "12|23|32": "M_24", "12|31|23": "M_25",
                 "12|23|31": "M_26", "12|32|31": "M_46", "12|21|21": "M_56", "12|21|12": "M_65",
                 "12|12|21": "M_66", "12|13|23": "12|13|23"}.items():
        assert tm.label_for_signature(s) == l


def test_merge_census_rules(tm, oracle):
    z = tm.merge_census(tm.StarCounter(), tm.PairCounter(), tm.TriCounter())
    assert z.total() == 0
    p = tm.PairCounter()
    p.cells[tm.PairCounter.index(O_, O_, O_)] = 5
    p.cells[tm.PairCounter.index(IN_, IN_, IN_)] = 5
    assert tm.merge_census(tm.StarCounter(), p, tm.TriCounter()).count("12|12|12") == 5
    p.cells[tm.PairCounter.index(IN_, IN_, IN_)] = 4
    with pytest.raises(tm.ConsistencyError):
        tm.merge_census(tm.StarCounter(), p, tm.TriCounter())
    t = tm.TriCounter()
    for idx in (tm.TriCounter.index(2, O_, IN_, O_), tm.TriCounter.index(1, IN_, O_, IN_),
                tm.TriCounter.index(0, O_, IN_, O_)):
        t.cells[idx] = 4
    assert tm.merge_census(tm.StarCounter(), tm.PairCounter(), t).count("12|31|23") == 4
    assert tm.merge_census(tm.StarCounter(), tm.PairCounter(), t, tm.TriangleMode.removal).count("12|31|23") == 12
    t2 = tm.TriCounter()
    t2.cells[tm.TriCounter.index(2, O_, O_, O_)] = 2
    with pytest.raises(tm.ConsistencyError):
        tm.merge_census(tm.StarCounter(), tm.PairCounter(), t2)
    tm.merge_census(tm.StarCounter(), tm.PairCounter(), t2, tm.TriangleMode.removal)
    # against the oracle's merge on random valid counters (linearity included)
    rng = np.random.default_rng(99)
    for _ in range(20):
        st = rng.integers(0, 1000, 24).astype(np.uint64)
        pr = rng.integers(0, 1000, 8).astype(np.uint64)
        pr[4:] = pr[:4][::-1]
        cls = [oracle.cell_signature(2, c) for c in range(24)]
        vals = {k: int(rng.integers(0, 100)) for k in set(cls)}
        tr = np.array([vals[c] for c in cls], np.uint64)
        got = tm.merge_census(tm.StarCounter(st), tm.PairCounter(pr), tm.TriCounter(tr)).counts
        assert (got == oracle.merge_census(st, pr, tr)).all()


def test_merge_overflow(tm):
    s = tm.StarCounter()
    s.cells[0] = np.uint64(2 ** 64 - 1)
    s.cells[1] = np.uint64(0)
    ok = tm.merge_census(s, tm.PairCounter(), tm.TriCounter())
    assert ok.count_at(ok.counts.argmax()) == 2 ** 64 - 1
    a = tm.StarCounter(); a.cells[0] = np.uint64(2 ** 64 - 1)
    b = tm.StarCounter(); b.cells[0] = 1
    with pytest.raises(tm.CounterOverflowError):
        a.add(b)


def test_generator_matches_reference(tm, oracle):
    for case in load_golden("random_reference.json")["cases"][:10]:
        g = tm.generate_random_graph(case["nodes"], case["edges"], case["t_max"], case["seed"])
        s, d, t = oracle.generate_random_graph(case["nodes"], case["edges"], case["t_max"], case["seed"])
        assert (g.src == s).all() and (g.dst == d).all() and (g.t == t).all()
    g = tm.generate_random_graph(2, 10, 100, 1)
    assert ((g.src < 2) & (g.dst < 2) & (g.src != g.dst)).all()
    assert tm.generate_random_graph(5, 0, 100, 42).edge_count() == 0
    with pytest.raises(ValueError):
        tm.generate_random_graph(1, 5, 100, 1)


def test_parse_edge_list(tm):
    g = tm.parse_edge_list("a c 4\na c 8\nd a 9\n")
    assert g.node_count() == 3 and g.edge_count() == 3
    assert [g.find_node(x) for x in "acd"] == [0, 1, 2] and g.find_node("z") is None
    g = tm.parse_edge_list("# header comment\n\na b 5 extra tokens here\r\n  \nb c 6\r\n")
    assert g.node_count() == 3 and g.edge_count() == 2 and int(g.t[0]) == 5
    g = tm.parse_edge_list("a a 5\na b 6\n")
    assert g.node_count() == 2 and g.edge_count() == 1 and g.dropped_self_loops() == 1
    with pytest.raises(tm.ParseError):
        tm.parse_edge_list("a a 5\n", drop_self_loops=False)
    g = tm.parse_edge_list("q q 1\na b 2\n")
    assert g.node_count() == 2 and g.find_node("q") is None
    with pytest.raises(tm.ParseError) as e:
        tm.parse_edge_list("a b 1\nc d xyz\n")
    assert e.value.line == 2 and "xyz" in str(e.value)
    with pytest.raises(tm.ParseError):
        tm.parse_edge_list("a b\n")
    assert tm.parse_edge_list("").edge_count() == 0
    g = tm.parse_edge_list("a b 5\nc b 5\nx y 1\n")
    s, d, t, o = g.edges()
    assert t.tolist() == [1, 5, 5] and o.tolist() == [2, 0, 1]
    # round trip
    g = tm.generate_random_graph(20, 200, 1000, 3)
    back = tm.parse_edge_list(tm.write_edge_list(g))
    s1, d1, t1, _ = g.edges(); s2, d2, t2, _ = back.edges()
    assert [g.node_id(int(x)) for x in s1] == [back.node_id(int(x)) for x in s2]
    assert (t1 == t2).all()


def test_partition_bounds_host_logic():
    from paper_2204_09236_b200.distributed import partition_bounds
    cp = np.concatenate([[0], np.cumsum(np.array([5, 1, 1, 1, 9, 1, 1, 1, 1, 1], np.uint64))])
    for world in (1, 2, 3, 4, 16):
        b = partition_bounds(cp, world)
        assert b[0][0] == 0 and b[-1][1] == 10 and len(b) == world
        for (x, y), (x2, _) in zip(b, b[1:]):
            assert y == x2 and x <= y


def test_parse_mirror_matches_reference_parser(tm):
    """The host mirror of parse_edge_list against the reference's own parser
    (oracle/_ref) on seeded fuzz texts, valid and with one planted error."""
    from oracle import Reference
    if not Reference.available():
        pytest.skip("reference build absent")
    from edgelist_fuzz import fuzz_text
    R = Reference()
    for seed in range(12):
        for err in ("", "short", "time", "loop"):
            text = fuzz_text(seed, 200, err)
            for drop in (True, False):
                try:
                    want = R.parse_edge_list(text.encode(), drop)
                except ValueError as e:
                    line, msg = e.args[0]
                    with pytest.raises(tm.ParseError) as got:
                        tm.parse_edge_list(text, drop)
                    assert got.value.line == line and str(got.value) == msg
                    continue
                g = tm.parse_edge_list(text, drop)
                names, s, d, t, dropped = want
                assert g.node_ids == names
                assert (g.src == s).all() and (g.dst == d).all() and (g.t == t).all()
                assert g.dropped_self_loops() == dropped
