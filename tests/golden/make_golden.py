"""Generate tests/golden/*.json from the reference itself (run in the build
container, where /root/reference exists).

  toy.txt               the Fig.-1 toy edge list (reference proj/tests/data/toy.txt)
  toy_frozen.json       the reference's frozen toy census (proj/tests/test_util.hpp:116-131)
  toy_reference.json    reference counters / census / per-center cells on the toy graph
  random_reference.json reference counters + census on seeded generate_random_graph inputs
                        (the SPEC acceptance sweep shapes: nodes 5..60, edges 10..600,
                        t in [0, 1e4], delta in {1, 10, 100, 1000}) plus tie-heavy cases
  uniform_reference.json reference census for BASELINE config 0
                        (10k nodes, 200k edges, t uniform in [0, 1e6), delta 1000)
  powerlaw_reference.json reference census for BASELINE config 1 (optional, slow)
  hubstress_reference.json reference census for BASELINE config 2 (100k nodes,
                        50M edges, delta 3600; numpy generator; optional, slow)

  powerlaw_deltas_reference.json reference census of config 1's input at delta
                        600 and 86400 (optional, slow)
  config4_slices_reference.json reference census of contiguous 10M-edge index
                        (= time) slices of config 4 (powerlaw_50m_600m, counter-based
                        generator synth.power_law_hashed, one early and one
                        mid-stream) at delta 600 / 3600 / 86400 (optional, slow)
  triadic_reference.json reference census of config 3 (triadic_25m_100m, synth.
                        triadic_hashed) at FULL size, delta 3600 and 86400 (optional, slow)
  config4_full_reference.json reference census of config 4 (600M edges) at FULL size,
                        delta 600 (optional; ~100 GB of host memory: run on the GPU box's host)

Usage: python tests/golden/make_golden.py [--powerlaw] [--hubstress] [--powerlaw-deltas]
          [--config4-slices] [--triadic] [--config4-full] [--only-extra]
"""
from __future__ import annotations

import hashlib
import json
import os
import re
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
REF_TESTS = "/root/reference/proj/tests"

from oracle import Reference  # noqa: E402


def edge_hash(src, dst, t) -> str:
    h = hashlib.sha256()
    for a in (src, dst, t):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()[:16]


def parse_toy(text):
    ids, index, src, dst, t = [], {}, [], [], []
    for line in text.splitlines():
        f = line.split()
        if not f or f[0].startswith("#"):
            continue
        for tok in f[:2]:
            if tok not in index:
                index[tok] = len(ids)
                ids.append(tok)
        src.append(index[f[0]]); dst.append(index[f[1]]); t.append(int(f[2]))
    return ids, np.array(src, np.uint32), np.array(dst, np.uint32), np.array(t, np.int64)


def counters(R, g, delta):
    st, pr, tr = R.counters(g, delta, removal=False)
    _, _, trr = R.counters(g, delta, removal=True)
    return {"star": [int(x) for x in st], "pair": [int(x) for x in pr],
            "tri_countall": [int(x) for x in tr], "tri_removal": [int(x) for x in trr]}


def hubstress_golden(R):
    from paper_2204_09236_b200 import synth
    n, s, d, tt = synth.hub_stress()
    delta = 3600
    g = R.build_graph(n, s, d, tt)
    out = {"config": "hubstress_100k_50m", "nodes": n, "edges": int(len(s)), "hash": edge_hash(s, d, tt),
           "delta": delta, "census": [int(x) for x in R.run_parallel(g, delta, os.cpu_count() or 1)]}
    R.free(g)
    json.dump(out, open(os.path.join(HERE, "hubstress_reference.json"), "w"))


def powerlaw_deltas_golden(R, deltas=(600, 86400)):
    """config 1's input at further deltas (the BASELINE delta sweep)."""
    from paper_2204_09236_b200 import synth
    n, s, d, tt = synth.power_law()
    g = R.build_graph(n, s, d, tt)
    out = {"config": "powerlaw_1m_10m", "nodes": n, "edges": int(len(s)), "hash": edge_hash(s, d, tt),
           "cases": []}
    for delta in deltas:
        out["cases"].append({"delta": delta,
                             "census": [int(x) for x in R.run_parallel(g, delta, os.cpu_count() or 1)]})
        json.dump(out, open(os.path.join(HERE, "powerlaw_deltas_reference.json"), "w"))
    R.free(g)


CONFIG4 = dict(n=50_000_000, m=600_000_000, mean_gap=0.05, seed=2204)
CONFIG4_SLICES = ((0, 10_000_000), (300_000_000, 310_000_000))
CONFIG3 = dict(n=25_000_000, m=100_000_000, closure=0.30, delta=86_400, mean_gap=1.0, seed=2204)


def _dump(out, name):
    tmp = os.path.join(HERE, name + ".tmp")
    json.dump(out, open(tmp, "w"))
    os.replace(tmp, os.path.join(HERE, name))


def config4_slices_golden(R, deltas=(600, 3600, 86400)):
    """Reference run_parallel (all host threads) on contiguous edge-index
    slices of config 4; the input is time-ordered, so an index slice is a
    time slice.  Node ids are kept (n = 50M)."""
    import time
    from paper_2204_09236_b200 import synth
    name = "config4_slices_reference.json"
    path = os.path.join(HERE, name)
    out = json.load(open(path)) if os.path.exists(path) else {
        "config": "powerlaw_50m_600m", "generator": "synth.power_law_hashed", **CONFIG4, "slices": []}
    slices = CONFIG4_SLICES
    if os.environ.get("GOLDEN_SLICES"):  # e.g. "120000000:180000000" (with GOLDEN_DELTAS="600,3600")
        slices = tuple(tuple(int(x) for x in p.split(":")) for p in os.environ["GOLDEN_SLICES"].split(","))
    if os.environ.get("GOLDEN_DELTAS"):
        deltas = tuple(int(x) for x in os.environ["GOLDEN_DELTAS"].split(","))
    for lo, hi in slices:
        have = [s for s in out["slices"] if s["lo"] == lo and s["hi"] == hi]
        entry = have[0] if have else None
        done = {c["delta"] for c in entry["cases"]} if entry else set()
        if done >= set(deltas):
            continue
        n, s, d, tt = synth.power_law_hashed(CONFIG4["n"], CONFIG4["m"], CONFIG4["mean_gap"], CONFIG4["seed"],
                                             lo=lo, hi=hi)
        if entry is None:
            entry = {"lo": lo, "hi": hi, "hash": edge_hash(s, d, tt), "cases": []}
            out["slices"].append(entry)
        g = R.build_graph(n, s, d, tt)
        for delta in deltas:
            if delta in done:
                continue
            t0 = time.time()
            census = R.run_parallel(g, delta, os.cpu_count() or 1)
            entry["cases"].append({"delta": delta, "census": [int(x) for x in census],
                                   "cpu_s": round(time.time() - t0, 1), "threads": os.cpu_count()})
            _dump(out, name)
            print("config4 slice", lo, hi, "delta", delta, "done in", round(time.time() - t0, 1), "s", flush=True)
        R.free(g)


def config4_full_golden(R, deltas=(600,)):
    """Reference run_parallel on the WHOLE of config 4 (600M edges; ~100 GB of
    host memory for the reference's graph and indexes, so it runs on the GPU
    box's host: `python tests/golden/make_golden.py --only-extra --config4-full`,
    output written under gpurun_out/ and committed from there)."""
    import time
    from paper_2204_09236_b200 import synth
    name = "config4_full_reference.json"
    out_dir = os.environ.get("GOLDEN_OUT", HERE)
    need_gb = int(os.environ.get("GOLDEN_NEED_GB", "150"))  # never drive the box out of memory
    avail = [int(l.split()[1]) for l in open("/proc/meminfo") if l.startswith("MemAvailable")][0] >> 20
    if avail < need_gb:
        print("config4 full: only", avail, "GB of host memory available, need", need_gb, "- skipped", flush=True)
        return
    path = os.path.join(out_dir, name)
    t0 = time.time()
    try:
        import torch
        gpu = torch.cuda.is_available()
    except ImportError:
        gpu = False
    if gpu:  # the torch twin on the GPU makes the identical arrays in seconds
        n, s, d, tt = synth.power_law_hashed(CONFIG4["n"], CONFIG4["m"], CONFIG4["mean_gap"], CONFIG4["seed"],
                                             device="cuda")
        s, d, tt = (x.cpu().numpy() for x in (s, d, tt))
        s, d = s.view(np.uint32), d.view(np.uint32)
        torch.cuda.empty_cache()
    else:
        n, s, d, tt = synth.power_law_hashed(CONFIG4["n"], CONFIG4["m"], CONFIG4["mean_gap"], CONFIG4["seed"])
    h = edge_hash(s, d, tt)
    gen_s = round(time.time() - t0, 1)
    print("config4 full: generated + hashed in", gen_s, "s, hash", h, flush=True)
    out = json.load(open(path)) if os.path.exists(path) else {
        "config": "powerlaw_50m_600m", "generator": "synth.power_law_hashed", **CONFIG4, "edges": int(len(s)),
        "hash": h, "cases": []}
    assert out["hash"] == h
    t0 = time.time()
    g = R.build_graph(n, s, d, tt)
    del s, d, tt
    build_s = round(time.time() - t0, 1)
    print("config4 full: reference graph + indexes built in", build_s, "s", flush=True)
    done = {c["delta"] for c in out["cases"]}
    for delta in deltas:
        if delta in done:
            continue
        t0 = time.time()
        census = R.run_parallel(g, delta, os.cpu_count() or 1)
        out["cases"].append({"delta": delta, "census": [int(x) for x in census], "cpu_s": round(time.time() - t0, 1),
                             "threads": os.cpu_count(), "generate_s": gen_s, "build_s": build_s})
        tmp = path + ".tmp"
        json.dump(out, open(tmp, "w"))
        os.replace(tmp, path)
        print("config4 full delta", delta, "done in", out["cases"][-1]["cpu_s"], "s", flush=True)
    R.free(g)


def triadic_golden(R, deltas=(3600, 86400)):
    """Reference run_parallel on the whole of config 3 (100M edges)."""
    import time
    from paper_2204_09236_b200 import synth
    name = "triadic_reference.json"
    path = os.path.join(HERE, name)
    n, s, d, tt = synth.triadic_hashed(**CONFIG3)
    h = edge_hash(s, d, tt)
    out = json.load(open(path)) if os.path.exists(path) else {
        "config": "triadic_25m_100m", "generator": "synth.triadic_hashed", **CONFIG3, "edges": int(len(s)),
        "hash": h, "cases": []}
    assert out["hash"] == h
    done = {c["delta"] for c in out["cases"]}
    g = R.build_graph(n, s, d, tt)
    del s, d, tt
    for delta in deltas:
        if delta in done:
            continue
        t0 = time.time()
        census = R.run_parallel(g, delta, os.cpu_count() or 1)
        out["cases"].append({"delta": delta, "census": [int(x) for x in census],
                             "cpu_s": round(time.time() - t0, 1), "threads": os.cpu_count()})
        _dump(out, name)
        print("triadic delta", delta, "done in", round(time.time() - t0, 1), "s", flush=True)
    R.free(g)


def main(with_powerlaw: bool, with_hubstress: bool = False, only_extra: bool = False,
         with_pl_deltas: bool = False):
    R = Reference()
    if only_extra:
        if with_hubstress:
            hubstress_golden(R)
        if with_pl_deltas:
            powerlaw_deltas_golden(R)
        if "--config4-slices" in sys.argv:
            config4_slices_golden(R)
        if "--triadic" in sys.argv:
            triadic_golden(R)
        if "--config4-full" in sys.argv:
            ds = os.environ.get("GOLDEN_DELTAS")
            config4_full_golden(R, tuple(int(x) for x in ds.split(",")) if ds else (600,))
        return
    sigs = R.signatures()

    toy_text = open(os.path.join(REF_TESTS, "data", "toy.txt")).read()
    open(os.path.join(HERE, "toy.txt"), "w").write(toy_text)

    util = open(os.path.join(REF_TESTS, "test_util.hpp")).read()
    block = util[util.index("frozen_toy_census"):]
    frozen = {m.group(1): int(m.group(2)) for m in re.finditer(r'\{"([123|]{8})", (\d+)\}', block)}
    assert len(frozen) == 36
    json.dump({"source": "proj/tests/test_util.hpp frozen_toy_census (delta = 10)",
               "delta": 10, "census": frozen}, open(os.path.join(HERE, "toy_frozen.json"), "w"), indent=1)

    ids, src, dst, t = parse_toy(toy_text)
    g = R.build_graph(len(ids), src, dst, t)
    toy = {"node_ids": ids, "signatures": sigs, "cases": []}
    for delta in (0, 1, 5, 10, 100):
        case = {"delta": delta, **counters(R, g, delta),
                "census": [int(x) for x in R.run_parallel(g, delta, 1)],
                "oracle_census": [int(x) for x in R.oracle_census(g, delta)],
                "per_center": []}
        for u in range(len(ids)):
            s = int(np.sum(src == u) + np.sum(dst == u))
            st, pr = R.star_pair_at_center(g, u, delta, 0, max(s - 2, 0))
            tr = R.triangles_at_center(g, u, delta, 0, max(s - 1, 0))
            case["per_center"].append({"node": u, "degree": s, "star": [int(x) for x in st],
                                       "pair": [int(x) for x in pr], "tri": [int(x) for x in tr]})
        toy["cases"].append(case)
    R.free(g)
    json.dump(toy, open(os.path.join(HERE, "toy_reference.json"), "w"))

    rng = np.random.default_rng(20220419)
    cases = []
    for k in range(48):
        n = int(rng.integers(5, 61)); m = int(rng.integers(10, 601))
        t_max = 10_000 if k % 4 else int(rng.integers(5, 60))  # every 4th case: heavy timestamp ties
        seed = int(rng.integers(1, 2 ** 31))
        s, d, tt = R.generate_random_graph(n, m, t_max, seed)
        g = R.build_graph(n, s, d, tt)
        entry = {"nodes": n, "edges": m, "t_max": t_max, "seed": seed, "hash": edge_hash(s, d, tt),
                 "auto_threshold": R.auto_degree_threshold(g), "deltas": []}
        for delta in (0, 1, 10, 100, 1000):
            entry["deltas"].append({"delta": delta, **counters(R, g, delta),
                                    "census": [int(x) for x in R.run_parallel(g, delta, 4)],
                                    "census_removal": [int(x) for x in R.run_parallel(g, delta, 1, -1, True)]})
        R.free(g)
        cases.append(entry)
    json.dump({"signatures": sigs, "cases": cases}, open(os.path.join(HERE, "random_reference.json"), "w"))

    # BASELINE config 0 (same generator as the reference)
    n, m, t_max, seed, delta = 10_000, 200_000, 999_999, 2204, 1000
    s, d, tt = R.generate_random_graph(n, m, t_max, seed)
    g = R.build_graph(n, s, d, tt)
    out = {"config": "uniform_10k_200k", "nodes": n, "edges": m, "t_max": t_max, "seed": seed,
           "hash": edge_hash(s, d, tt), "delta": delta, **counters(R, g, delta),
           "census": [int(x) for x in R.run_parallel(g, delta, os.cpu_count() or 1)]}
    R.free(g)
    json.dump(out, open(os.path.join(HERE, "uniform_reference.json"), "w"))

    if with_powerlaw:
        from paper_2204_09236_b200 import synth
        n, s, d, tt = synth.power_law()
        delta = 3600
        g = R.build_graph(n, s, d, tt)
        out = {"config": "powerlaw_1m_10m", "nodes": n, "edges": int(len(s)), "hash": edge_hash(s, d, tt),
               "delta": delta, "census": [int(x) for x in R.run_parallel(g, delta, os.cpu_count() or 1)]}
        R.free(g)
        json.dump(out, open(os.path.join(HERE, "powerlaw_reference.json"), "w"))
    if with_hubstress:
        hubstress_golden(R)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main("--powerlaw" in sys.argv, "--hubstress" in sys.argv, "--only-extra" in sys.argv,
         "--powerlaw-deltas" in sys.argv)
