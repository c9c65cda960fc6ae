"""CPU: the oracle (plain-C restatement, oracle/tmotif_oracle.c) pinned to the
reference's golden vectors and, when present, to the reference itself."""
import hashlib

import numpy as np
import pytest

from conftest import load_golden, toy_arrays


def edge_hash(src, dst, t):
    h = hashlib.sha256()
    for a in (src, dst, t):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()[:16]


def test_signatures_match_reference(oracle):
    assert oracle.signatures() == load_golden("random_reference.json")["signatures"]
    assert oracle.signatures() == load_golden("toy_reference.json")["signatures"]


def test_toy_frozen_census(oracle):
    """test_oracle.cpp:117-124 frozen toy census, via brute force AND FAST."""
    frozen = load_golden("toy_frozen.json")["census"]
    sigs = oracle.signatures()
    g = toy_arrays()
    og = oracle.build_graph(g.node_count(), g.src, g.dst, g.t)
    bf = oracle.census_bruteforce(og, 10)
    fast = oracle.census(og, 10)
    for k, s in enumerate(sigs):
        assert bf[k] == frozen[s], s
        assert fast[k] == frozen[s], s


def test_toy_reference_counters(oracle):
    ref = load_golden("toy_reference.json")
    g = toy_arrays()
    og = oracle.build_graph(g.node_count(), g.src, g.dst, g.t)
    for case in ref["cases"]:
        d = case["delta"]
        st, pr = oracle.count_star_pair(og, d)
        assert st.tolist() == case["star"] and pr.tolist() == case["pair"]
        assert oracle.count_triangles(og, d).tolist() == case["tri_countall"]
        assert oracle.count_triangles(og, d, True).tolist() == case["tri_removal"]
        assert oracle.census(og, d).tolist() == case["census"]
        assert oracle.census_bruteforce(og, d).tolist() == case["oracle_census"]
        for pc in case["per_center"]:
            s = pc["degree"]
            st, pr = oracle.star_pair_at_center(og, pc["node"], d, 0, max(s - 2, 0))
            assert st.tolist() == pc["star"] and pr.tolist() == pc["pair"]
            assert oracle.triangles_at_center(og, pc["node"], d, 0, max(s - 1, 0)).tolist() == pc["tri"]


def test_random_sweep_matches_reference(oracle):
    gold = load_golden("random_reference.json")
    for case in gold["cases"]:
        s, d, t = oracle.generate_random_graph(case["nodes"], case["edges"], case["t_max"], case["seed"])
        assert edge_hash(s, d, t) == case["hash"]
        og = oracle.build_graph(case["nodes"], s, d, t)
        assert oracle.auto_degree_threshold(og) == case["auto_threshold"]
        for dc in case["deltas"]:
            delta = dc["delta"]
            st, pr = oracle.count_star_pair(og, delta)
            assert st.tolist() == dc["star"] and pr.tolist() == dc["pair"]
            tri = oracle.count_triangles(og, delta)
            trr = oracle.count_triangles(og, delta, True)
            assert tri.tolist() == dc["tri_countall"] and trr.tolist() == dc["tri_removal"]
            assert oracle.merge_census(st, pr, tri).tolist() == dc["census"]
            assert oracle.merge_census(st, pr, trr, True).tolist() == dc["census_removal"]
        oracle.free(og)


def test_fast_equals_bruteforce(oracle):
    """SPEC acceptance 1 (oracle equivalence) on the restatement itself."""
    rng = np.random.default_rng(1)
    for k in range(40):
        n = int(rng.integers(5, 40)); m = int(rng.integers(10, 300))
        s, d, t = oracle.generate_random_graph(n, m, 10_000 if k % 3 else 30, int(rng.integers(1, 1 << 30)))
        og = oracle.build_graph(n, s, d, t)
        for delta in (1, 10, 100, 1000):
            assert (oracle.census(og, delta) == oracle.census_bruteforce(og, delta)).all()
            assert (oracle.census(og, delta, True) == oracle.census(og, delta)).all()
        oracle.free(og)


def test_config0_uniform_matches_reference(oracle):
    ref = load_golden("uniform_reference.json")
    s, d, t = oracle.generate_random_graph(ref["nodes"], ref["edges"], ref["t_max"], ref["seed"])
    assert edge_hash(s, d, t) == ref["hash"]
    og = oracle.build_graph(ref["nodes"], s, d, t)
    st, pr = oracle.count_star_pair(og, ref["delta"])
    assert st.tolist() == ref["star"] and pr.tolist() == ref["pair"]
    assert oracle.count_triangles(og, ref["delta"]).tolist() == ref["tri_countall"]
    assert oracle.census(og, ref["delta"]).tolist() == ref["census"]


def test_restatement_against_live_reference(oracle):
    from oracle import Reference
    if not Reference.available():
        pytest.skip("oracle/_ref not built (reference tree absent)")
    R = Reference()
    rng = np.random.default_rng(77)
    for k in range(12):
        n = int(rng.integers(3, 30)); m = int(rng.integers(0, 400))
        s, d, t = R.generate_random_graph(n, m, int(rng.integers(1, 5000)), int(rng.integers(1, 1 << 30)))
        og = oracle.build_graph(n, s, d, t); rg = R.build_graph(n, s, d, t)
        for delta in (0, 5, 77, 4000):
            st, pr, tr = R.counters(rg, delta)
            st2, pr2 = oracle.count_star_pair(og, delta)
            assert (st == st2).all() and (pr == pr2).all()
            assert (tr == oracle.count_triangles(og, delta)).all()
        oracle.free(og); R.free(rg)
