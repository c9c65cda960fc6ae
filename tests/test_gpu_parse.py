"""GPU edge-list reader (tm_parse_edge_list) against the reference's own
parse_edge_list (oracle/_ref, graph.cpp:73-116) -- the reference's
test_graph.cpp cases, seeded fuzz texts with every construct the reader
distinguishes, each error kind (line number and message), device-resident
text, and a 2M-line text whose census is counted straight from the parsed
device arrays."""
import numpy as np
import pytest

from edgelist_fuzz import fuzz_text

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ref():
    from oracle import Reference
    if not Reference.available():
        pytest.skip("reference build absent")
    return Reference()


def gpu_parse(tm, text, drop=True):
    el = tm.parse_edge_list_gpu(text, drop)
    g = el.to_graph()
    el.close()
    return g


def check_same(tm, ref, text: str, drop=True):
    try:
        want = ref.parse_edge_list(text.encode(), drop)
    except ValueError as e:
        line, msg = e.args[0]
        with pytest.raises(tm.ParseError) as got:
            gpu_parse(tm, text, drop)
        assert got.value.line == line and str(got.value) == msg, (got.value.line, str(got.value), line, msg)
        return None
    g = gpu_parse(tm, text, drop)
    names, s, d, t, dropped = want
    assert g.node_ids == names
    assert (g.src == s).all() and (g.dst == d).all() and (g.t == t).all()
    assert g.dropped_self_loops() == dropped
    return g


def test_reference_test_graph_cases(cuda, tm, ref):
    """test_graph.cpp:11-86."""
    g = check_same(tm, ref, "a c 4\na c 8\nd a 9\n")
    assert g.node_count() == 3 and g.find_node("a") == 0 and g.find_node("c") == 1 and g.find_node("d") == 2
    g = check_same(tm, ref, "# header comment\n\na b 5 extra tokens here\r\n  \nb c 6\r\n")
    assert g.node_count() == 3 and g.edge_count() == 2 and g.t[0] == 5
    g = check_same(tm, ref, "a a 5\na b 6\n")
    assert g.node_count() == 2 and g.edge_count() == 1 and g.dropped_self_loops() == 1
    with pytest.raises(tm.ParseError):
        gpu_parse(tm, "a a 5\n", drop=False)
    g = check_same(tm, ref, "q q 1\na b 2\n")
    assert g.find_node("q") is None
    with pytest.raises(tm.ParseError) as e:
        gpu_parse(tm, "a b 1\nc d xyz\n")
    assert e.value.line == 2 and "xyz" in str(e.value)
    with pytest.raises(tm.ParseError):
        gpu_parse(tm, "a b\n")
    g = check_same(tm, ref, "")
    assert g.node_count() == 0 and g.edge_count() == 0
    check_same(tm, ref, "a b 5\nc b 5\nx y 1\n")
    toy = open(__import__("os").path.join(__import__("conftest").GOLDEN, "toy.txt")).read()
    g = check_same(tm, ref, toy)
    assert g.node_count() == 5 and g.edge_count() == 12


def test_edge_constructs(cuda, tm, ref):
    for text in ["a b 1", "a b 1\n", "\n\n\n", "#only\n# comments", "  \t \r\n", "a\tb\v7\f\r\n",
                 "x y -9223372036854775808\ny x 9223372036854775807\n", "a b 9223372036854775808\n",
                 "a b -\n", "a b +1\n", "a # 3\n#a b 3\n", "é λ 3\nλ é 4\n", "a b 1 2 3 4 5 6\n",
                 "a b 1\na b\n", "a a x\n", "a b x\nc c 1\n", "aa a 1\na aa 2\n", "a b 00012\n",
                 "a b 1\r\r\n", " a b 1\n"]:
        for drop in (True, False):
            check_same(tm, ref, text, drop)


def test_fuzz_against_reference(cuda, tm, ref):
    for seed in range(40):
        for err in ("", "short", "time", "loop"):
            text = fuzz_text(1000 + seed, 600, err)
            for drop in (True, False):
                check_same(tm, ref, text, drop)


def test_long_lines_and_many_blocks(cuda, tm, ref):
    """Lines longer than a block's shared-memory stage (global fallback) and
    texts spanning many line blocks."""
    rng = np.random.default_rng(5)
    lines = []
    for i in range(3000):
        if i % 97 == 0:
            lines.append("#" + "x" * 40000)
        elif i % 101 == 0:
            lines.append("n%d m%d %d %s" % (i, i + 1, i, "pad " * 10000))
        else:
            lines.append("v%d w%d %d" % (rng.integers(500), rng.integers(500) + 500, rng.integers(10 ** 9)))
    check_same(tm, ref, "\n".join(lines))


def test_device_text_and_census_from_parsed_arrays(cuda, tm, oracle):
    """2M edges written as text (ids renamed), parsed from DEVICE memory, and
    counted from the parsed device arrays: the census equals the one of the
    original arrays (the renaming is a relabelling)."""
    import torch
    n, m, delta = 200_000, 2_000_000, 5000
    s, d, t = oracle.generate_random_graph(n, m, 10 ** 7, 77)
    names = np.array(["node-%x" % (u * 2654435761 % (1 << 32)) for u in range(n)])
    text = "\n".join(f"{a} {b} {c}" for a, b, c in zip(names[s], names[d], t)).encode()
    dev = torch.frombuffer(bytearray(text), dtype=torch.uint8).cuda()
    el = tm.parse_edge_list_gpu((dev.data_ptr(), len(text)))
    assert el.m == m and el.dropped_self_loops == 0
    g = el.to_graph()
    # the parsed ids are a relabelling of the original ones
    lookup = {nm: i for i, nm in enumerate(g.node_ids)}
    relabel = np.array([lookup.get(nm, -1) for nm in names])
    assert (relabel[s] == g.src).all() and (relabel[d] == g.dst).all() and (g.t == t).all()
    ps, pd, pt = el.device_arrays()
    cfg = tm.RunConfig(delta=delta)
    got = tm.count_edges_device(g.node_count(), m, ps, pd, pt, cfg)
    ds = torch.from_numpy(s.view(np.int32)).cuda()
    dd = torch.from_numpy(d.view(np.int32)).cuda()
    dt = torch.from_numpy(t).cuda()
    want = tm.count_edges_device(n, m, ds.data_ptr(), dd.data_ptr(), dt.data_ptr(), cfg)
    assert got.tolist() == want.tolist()
    el.close()


def test_write_edge_list_round_trip(cuda, tm, oracle):
    """write_edge_list (graph.cpp:170) on the GPU for decimal ids equals the
    host writer byte for byte, and parses back to the same edges
    (test_graph.cpp 'write/parse round trip')."""
    s, d, t = oracle.generate_random_graph(20, 200, 1000, 3)
    t = t.copy()
    t[::7] = -t[::7]  # negative times format with a sign
    t[3] = -(2 ** 63)
    t[4] = 2 ** 63 - 1
    # the reference writes graph.edges(), i.e. (t, ordinal) order; the GPU
    # writer keeps the given order, so hand it the edges in that order
    o = np.argsort(t, kind="stable")
    s, d, t = s[o], d[o], t[o]
    g = tm.TemporalGraph([str(u) for u in range(20)], s, d, t)
    text = tm.write_edge_list_gpu(s, d, t)
    assert text.decode() == tm.write_edge_list(g)
    back = tm.parse_edge_list_gpu(text).to_graph()
    assert [back.node_ids[u] for u in back.src] == [str(u) for u in s]
    assert [back.node_ids[u] for u in back.dst] == [str(u) for u in d]
    assert (back.t == t).all()
    assert tm.write_edge_list_gpu(s[:0], d[:0], t[:0]) == b""


def test_many_distinct_tokens_regrow_table(cuda, tm):
    """3M distinct tokens: more than the first interning table takes, so the
    table is regrown; ids stay in first-appearance order (u0 v0 u1 v1 ...)."""
    k = 1_500_000
    text = "".join(f"u{i} v{i} {i}\n" for i in range(k))
    g = tm.parse_edge_list_gpu(text).to_graph()
    assert g.node_count() == 2 * k and g.edge_count() == k
    assert (g.src == np.arange(0, 2 * k, 2)).all() and (g.dst == np.arange(1, 2 * k, 2)).all()
    assert g.node_ids[:4] == ["u0", "v0", "u1", "v1"] and g.node_ids[-1] == f"v{k - 1}"
    assert (g.t == np.arange(k)).all()
    # long tokens (> 7 bytes: hashed keys with byte compares), repeated
    text = "".join(f"longnode-{i % 1000:06d} other-node-{i % 777:05d} {i}\n" for i in range(200_000))
    g = tm.parse_edge_list_gpu(text).to_graph()
    assert g.node_count() == 1777
    assert g.node_ids[g.src[12345]] == f"longnode-{12345 % 1000:06d}"
    assert g.node_ids[g.dst[12345]] == f"other-node-{12345 % 777:05d}"
