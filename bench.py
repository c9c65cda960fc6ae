"""bench.py -- exact 36-motif temporal census throughput on B200.

Step = one full census of the BASELINE workload from edge arrays resident in
HBM: GPU index build (radix sorts -> S / G / F layouts) + FAST-Star pass +
FAST-Tri pass + counter all-reduce (N > 1) + merge.  value = edges x steps /
max-over-ranks device time.  e2e = the same step through the C-ABI from
pinned HOST arrays, host->device copies and the counter read-back inside the
timed region.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config NAME] [--impl ours|reference]

--impl reference times the reference's own CPU implementation (oracle/_ref:
the unmodified reference sources, std::thread HARE executor with all host
threads) on a bounded time slice of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

MEASURED_PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")
METRIC = "temporal edges/sec, exact 36-motif count (1/2/4/8 B200); % of HBM roofline"

# Algorithmic bytes per STEP for each kernel family that can dominate a step
# (DESIGN.md "Roofline"): bytes that must cross HBM at least once.
#   star_filter   per edge: P t (8 B) + w (4 B), neighbours' t from the same lines
#   gather_s      per incident record: sorted key 8 B + edge record 8 B (16 B when the
#                 time span needs more than 32 bits) + S outputs 20 B
#   gather_p      per edge: sorted key 8 B + edge record 8/16 B + P outputs 24 B
#   tri_filter    per forward record (one per edge): F t (8 B) + node (4 B)
#   star_work / tri_work run on the filtered worklists only (random access, no streaming model)
#   radix_downsweep per key per digit pass: key (+ value) read + write
#                 node sort: packed u64 keys over 2m records, ceil(nb/8) passes
#                 pair sort: packed u64 keys (min << 32 | edge) over m edges, ceil(nb/8) passes
#                 t sort:    packed u64 keys over m edges, ceil(tbits/8) passes (unsorted input only)
#   scan          per element: predicate inputs read (4 B) + u32 output written (4 B)
def algo_bytes(n, m, t):
    R = 2 * m
    nb = max(1, int(n - 1).bit_length())
    pbits = max(1, int(m - 1).bit_length())
    tb = int(int(t.max()) - int(t.min())).bit_length() if m else 0
    unsorted = bool(m > 1 and (np.diff(t) < 0).any())
    # node sort: packed u64 keys (node << 32 | record), keys only
    sort = R * 8 * 2 * ((nb + 7) // 8)
    # pair sort: the max-side records re-sorted by the min endpoint, keys only
    sort += m * 8 * 2 * ((nb + 7) // 8)
    if unsorted:
        sort += m * (8 if tb + pbits <= 64 else 12) * 2 * ((tb + 7) // 8)
    eb = 8 if tb <= 32 else 16  # narrow / wide edge records (tm_graph.cu EdgeCodec)
    return {"star_filter": m * 12, "tri_filter": m * 12, "radix_downsweep": sort,
            "gather_s": R * (8 + eb + 20), "gather_p": m * (8 + eb + 24), "scan": 2 * R * 4 + m * 8}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def load_workload(name: str, delta=None):
    from paper_2204_09236_b200 import synth
    if name in synth.CONFIGS:
        cfg = synth.CONFIGS[name]
        n, src, dst, t = cfg["fn"]()
        return n, src, dst, t, int(delta if delta is not None else cfg["delta"])
    cfg = synth.GPU_CONFIGS[name]  # generated on the GPU, copied to host arrays
    n, src, dst, t = cfg["fn"]()
    d = delta if delta is not None else cfg.get("delta", (cfg.get("deltas") or [3600])[1 if len(cfg.get("deltas", [])) > 1 else 0])
    out = (src.cpu().numpy().view(np.uint32), dst.cpu().numpy().view(np.uint32), t.cpu().numpy())
    del src, dst, t
    import torch
    torch.cuda.empty_cache()
    return n, out[0], out[1], out[2], int(d)


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.lines = []
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()
                out = ""
            self.lines = [l for l in out.splitlines() if l.strip()]

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in getattr(self, "lines", []):
            f = [x.strip() for x in l.split(",")]
            try:
                sm.append(float(f[0]))
                mx = max(mx, float(f[1]))
            except (ValueError, IndexError):
                continue
            for nm, v in zip(names, f[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def peaks():
    try:
        with open(MEASURED_PEAKS) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def cpu_reference(n, src, dst, t, delta, steps, warmup, sample_edges, threads):
    """Time the reference's own pipeline (TemporalGraph::build + GraphContext::build
    + run_parallel) on the first `sample_edges` edges in time order."""
    from oracle import Reference
    R = Reference()
    order = np.argsort(t, kind="stable")[:sample_edges]
    order.sort()  # keep ingestion order of the slice
    s, d, tt = src[order], dst[order], t[order]
    times = []
    census = None
    for i in range(warmup + steps):
        t0 = time.perf_counter()
        census, mb, mc = R.pipeline(n, s, d, tt, delta, threads)
        dt = time.perf_counter() - t0
        if i >= warmup:
            times.append(dt)
    sec = float(np.mean(times))
    return {"value": len(s) / sec, "sec_per_step": sec, "edges": int(len(s)), "census_total": int(census.sum())}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="powerlaw_1m_10m")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-reader", action="store_true", help="skip the edge-list reader measurement")
    ap.add_argument("--cpu-sample-edges", type=int, default=1_000_000)
    ap.add_argument("--delta", type=int, default=None, help="override the config's delta")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="counter all-reduce backend (gloo: CPU tensors, for multi-rank tests on one GPU)")
    ap.add_argument("--partition", default="time", choices=["time", "centers"],
                    help="N>1: time slices of the first edge (each rank indexes only its slice) or "
                         "center ranges over a replicated graph")
    ap.add_argument("--same-device", action="store_true",
                    help="testing only: every rank uses cuda:0 (independent kernels, gloo reduce)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    threads = os.cpu_count() or 1

    n, src, dst, t, delta = load_workload(args.config, args.delta)
    m = len(src)
    base_cfg = {"workload": args.config, "nodes": int(n), "edges": int(m), "delta": int(delta),
                "inputs": "time-ordered synthetic edge list (seed 2204), ingestion order = time order",
                "l2": "inputs + indexes (~1 GB) exceed the 126 MB L2; no explicit flush"}

    if args.impl == "reference":
        if rank != 0:
            return
        res = cpu_reference(n, src, dst, t, delta, args.steps, args.warmup, min(args.cpu_sample_edges, m), threads)
        sample = f"first {res['edges']} of {m} edges in time order (a time slice of the same workload)"
        line = {"metric": METRIC, "value": res["value"], "unit": "edges/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": res["sec_per_step"] * 1e3, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "int64", "data": "synthetic",
                "impl": "reference",
                "config": dict(base_cfg, parallelism="cpu", sample=sample),
                "cpu_baseline": {"value": res["value"], "unit": "edges/s", "cores": threads, "kind": "reference",
                                 "sample": sample},
                "e2e": {"value": res["value"], "unit": "edges/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    import torch
    if args.same_device:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    red_dev = dev if args.dist_backend == "nccl" else torch.device("cpu")
    dist = None
    if world > 1:
        import torch.distributed as dist
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")
    import paper_2204_09236_b200 as tm

    stream = torch.cuda.Stream(device=dev)
    sptr = stream.cuda_stream
    cfg = tm.RunConfig(delta=delta)
    center = (0, 0)
    if world > 1 and args.partition == "time":
        # each rank holds the edges with t in [lo, hi + delta) and owns the
        # instances whose earliest edge has t in [lo, hi): exact partition
        from paper_2204_09236_b200.distributed import time_slice_bounds, time_slice_mask
        lo, hi = time_slice_bounds(t, world)[rank]
        keep = time_slice_mask(t, lo, hi, delta)
        src, dst, t = src[keep], dst[keep], t[keep]
        cfg = tm.RunConfig(delta=delta, first_edge_t_end=hi)
    m_local = len(src)
    # inputs resident in HBM
    d_src = torch.from_numpy(src.view(np.int32)).to(dev)
    d_dst = torch.from_numpy(dst.view(np.int32)).to(dev)
    d_t = torch.from_numpy(t).to(dev)
    # pinned host copies for the e2e leg
    h_src = torch.from_numpy(src.view(np.int32)).pin_memory()
    h_dst = torch.from_numpy(dst.view(np.int32)).pin_memory()
    h_t = torch.from_numpy(t).pin_memory()
    torch.cuda.synchronize()
    if world > 1 and args.partition == "centers":
        ctx = tm.GraphContext.build_device(n, d_src.data_ptr(), d_dst.data_ptr(), d_t.data_ptr(), m_local,
                                           stream=sptr)
        center = ctx.partition(world, rank)
        ctx.close()
    red = torch.zeros(56, dtype=torch.int64, device=red_dev)
    raw = np.zeros(56, np.uint64)

    def step(host: bool):
        if host:
            census = tm.count_edges(n, h_src.numpy().view(np.uint32), h_dst.numpy().view(np.uint32), h_t.numpy(),
                                    cfg, stream=sptr, raw_out=raw, center=center)
        else:
            census = tm.count_edges_device(n, m_local, d_src.data_ptr(), d_dst.data_ptr(), d_t.data_ptr(), cfg,
                                           stream=sptr, center=center, raw_out=raw)
        if world > 1:  # one all-reduce of the 56 raw u64 counters (exact modulo 2^64)
            with torch.cuda.stream(stream):
                red.copy_(torch.from_numpy(raw.view(np.int64)), non_blocking=False)
                dist.all_reduce(red)
                tot = red.cpu().numpy().view(np.uint64)
            census = tm.merge_census(tm.StarCounter(tot[:24]), tm.PairCounter(tot[24:32]), tm.TriCounter(tot[32:]),
                                     cfg.triangle_mode).counts
        return census

    def timed(host: bool, steps: int, warmup: int):
        for _ in range(warmup):
            census = step(host)
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        l0 = tm.kernel_launches()
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            ev0.record(stream)
        for _ in range(steps):
            census = step(host)
        with torch.cuda.stream(stream):
            ev1.record(stream)
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        ms = ev0.elapsed_time(ev1)
        if dist:
            x = torch.tensor([ms], dtype=torch.float64, device=red_dev)
            dist.all_reduce(x, op=dist.ReduceOp.MAX)
            ms = float(x.item())
        return ms / steps, census, tm.kernel_launches() - l0

    def reduce_raw(census):
        if world > 1:  # one all-reduce of the 56 raw u64 counters (exact modulo 2^64)
            with torch.cuda.stream(stream):
                red.copy_(torch.from_numpy(raw.view(np.int64)), non_blocking=False)
                dist.all_reduce(red)
                tot = red.cpu().numpy().view(np.uint64)
            census = tm.merge_census(tm.StarCounter(tot[:24]), tm.PairCounter(tot[24:32]), tm.TriCounter(tot[32:]),
                                     cfg.triangle_mode).counts
        return census

    def timed_pipelined(steps: int, warmup: int):
        """e2e through tm_count_edges_async: batch i+1's host->device copy overlaps
        batch i's census (two batches staged); every step still copies its
        inputs from pinned host memory and reads its counters back."""
        from collections import deque

        def submit():
            return tm.count_edges_async(n, h_src.numpy().view(np.uint32), h_dst.numpy().view(np.uint32),
                                        h_t.numpy(), cfg, stream=sptr)

        def collect(p):
            return reduce_raw(p.result(raw_out=raw))

        for _ in range(max(warmup, 4)):  # both staging slots: eager run, capture, replay
            census = collect(submit())
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            ev0.record(stream)
        q = deque()
        for _ in range(steps):
            q.append(submit())
            if len(q) > 1:
                census = collect(q.popleft())
        while q:
            census = collect(q.popleft())
        with torch.cuda.stream(stream):
            ev1.record(stream)
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        ms = ev0.elapsed_time(ev1)
        if dist:
            x = torch.tensor([ms], dtype=torch.float64, device=red_dev)
            dist.all_reduce(x, op=dist.ReduceOp.MAX)
            ms = float(x.item())
        return ms / steps, census

    with ClockSampler(local) as clk:
        ms_step, census, launches = timed(False, args.steps, args.warmup)
    ms_e2e_sync, census_e2e, _ = timed(True, max(2, args.steps // 2), args.warmup)
    assert (census == census_e2e).all(), "device and host paths disagree"
    e2e_api = "tm_count_edges_async (two batches in flight: copy of batch i+1 overlaps census i)"
    if tuple(center) == (0, 0):
        # >= 8 batches: the pipeline fill (first copy, last census) is amortised
        ms_e2e, census_pipe = timed_pipelined(max(8, args.steps), args.warmup)
        assert (census == census_pipe).all(), "device and pipelined host paths disagree"
    else:  # center ranges go through the synchronous API only
        ms_e2e = ms_e2e_sync
        e2e_api = "tm_count_edges (one batch at a time)"

    # per-kernel device time with CUDA events on the launching stream (separate instrumented pass)
    tm.kernel_timing(enable=True, reset=True)
    kk = max(2, min(args.steps, 5))
    for _ in range(kk):
        step(False)
    torch.cuda.synchronize()
    tm.kernel_timing(enable=False)
    names = ["star_filter", "star_work", "tri_filter", "tri_wedge", "tri_long", "radix_upsweep",
             "radix_downsweep", "radix_scan", "scan", "gather_s", "gather_p", "forward_scatter", "pack_edges", "pair_keys",
             "time_keys", "perm_from_keys", "validate", "offsets", "forward_off"]
    ktimes = {}
    for nm in names:
        tot_ms, cnt = tm.kernel_time(nm)
        if cnt:
            ktimes[nm] = {"ms_per_step": tot_ms / kk, "launches_per_step": cnt / kk}
    abytes = algo_bytes(n, m_local, t)
    dom = max(abytes, key=lambda k: ktimes.get(k, {}).get("ms_per_step", 0))
    dom_ms = ktimes[dom]["ms_per_step"]
    dom_launches = max(1.0, ktimes[dom]["launches_per_step"])
    algo = abytes[dom] / dom_launches
    launch_ms = dom_ms / dom_launches
    peak, peak_kind = peaks()
    achieved = algo / (launch_ms * 1e-3) / 1e9
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "r01", f"traffic_{dom}_{args.config}.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get("bytes_per_launch")
        except Exception:
            traffic = None
    for k, v in ktimes.items():
        if k in abytes:
            v["algo_GBps"] = abytes[k] / (v["ms_per_step"] * 1e-3) / 1e9

    # the edge-list reader in front of the path (N = 1): the same edges as
    # "SRC DST T" text, parsed on the GPU from device memory and from host
    # memory; the parsed arrays are counted once and must give the same census
    reader = None
    if world == 1 and not args.no_reader:
        nbytes = tm.write_edge_list_device(m_local, d_src.data_ptr(), d_dst.data_ptr(), d_t.data_ptr(), stream=sptr)
        d_text = torch.empty(nbytes + 16, dtype=torch.uint8, device=dev)
        tm.write_edge_list_device(m_local, d_src.data_ptr(), d_dst.data_ptr(), d_t.data_ptr(), d_text.data_ptr(),
                                  stream=sptr)
        h_text = d_text[:nbytes].cpu().pin_memory()
        torch.cuda.synchronize()
        el = tm.parse_edge_list_gpu((d_text.data_ptr(), nbytes), stream=sptr)
        assert el.m == m_local
        ps, pd, pt = el.device_arrays()
        census_txt = tm.count_edges_device(el.n, el.m, ps, pd, pt, cfg, stream=sptr)
        assert (census_txt == census).all(), "census of the parsed text differs"
        el.close()

        def time_parse(src_arg, reps=5):
            for _ in range(2):
                tm.parse_edge_list_gpu(src_arg, stream=sptr).close()
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(stream):
                e0.record(stream)
            for _ in range(reps):
                tm.parse_edge_list_gpu(src_arg, stream=sptr).close()
            with torch.cuda.stream(stream):
                e1.record(stream)
            torch.cuda.synchronize()
            return e0.elapsed_time(e1) / reps

        ms_dev = time_parse((d_text.data_ptr(), nbytes))
        ms_host = time_parse((h_text.data_ptr(), nbytes, False))
        reader = {"what": "tm_parse_edge_list: the reference's parse_edge_list (graph.cpp:73) on the GPU",
                  "text_bytes": int(nbytes), "lines": int(m_local),
                  "device_text": {"ms": ms_dev, "GB_per_s": nbytes / (ms_dev * 1e-3) / 1e9,
                                  "lines_per_s": m_local / (ms_dev * 1e-3)},
                  "host_text": {"ms": ms_host, "GB_per_s": nbytes / (ms_host * 1e-3) / 1e9,
                                "lines_per_s": m_local / (ms_host * 1e-3),
                                "note": "pinned host text, host->device copy inside the timed call"}}
        del d_text

    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return

    # reported CPU baseline: the reference's own code on host cores, rank 0, N = 1 only
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        try:
            from oracle import Reference
            if Reference.available():
                res = cpu_reference(n, src, dst, t, delta, 1, 0, min(args.cpu_sample_edges, m), threads)
                cpu = {"value": res["value"], "unit": "edges/s", "cores": threads, "kind": "reference",
                       "sample": f"first {res['edges']} of {m} edges in time order (one pipeline run: "
                                 f"build + run_parallel, {threads} std::threads)"}
        except Exception as ex:  # pragma: no cover
            log("cpu baseline failed:", ex)
        if reader is not None:
            try:  # the reference's own reader on a prefix of the same text
                from oracle import Reference
                if Reference.available():
                    k = min(args.cpu_sample_edges, m)
                    arr = h_text.numpy()[:nbytes]
                    cut = int(np.flatnonzero(arr == 10)[k - 1]) + 1
                    sample = bytes(arr[:cut])
                    t0 = time.perf_counter()
                    Reference().parse_edge_list(sample)
                    sec = time.perf_counter() - t0
                    reader["cpu_reference"] = {"lines_per_s": k / sec, "GB_per_s": len(sample) / sec / 1e9,
                                               "cores": 1, "kind": "reference",
                                               "sample": f"first {k} lines (parse_edge_list incl. TemporalGraph::build)"}
            except Exception as ex:  # pragma: no cover
                log("reader cpu baseline failed:", ex)

    value = m / (ms_step * 1e-3)
    line = {
        "metric": METRIC, "value": value, "unit": "edges/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "int64", "data": "synthetic",
        "config": dict(base_cfg, parallelism=("single GPU" if world == 1 else
                                              f"time slices of the first edge over {world} GPUs (each GPU indexes "
                                              f"its delta-extended slice)" if args.partition == "time" else
                                              f"center ranges over {world} GPUs, graph replicated")),
        "census_total": int(np.asarray(census, np.uint64).sum()),
        "e2e": {"value": m / (ms_e2e * 1e-3), "unit": "edges/s", "h2d_bytes_per_step": int(m_local * 16),
                "d2h_bytes_per_step": int(56 * 8 + 36 * 8), "ms_per_step": ms_e2e,
                "api": e2e_api,
                "sync_api": {"value": m / (ms_e2e_sync * 1e-3), "ms_per_step": ms_e2e_sync,
                             "api": "tm_count_edges (one batch at a time)"}},
        "gpu_launches": int(launches),
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "peak_kind": peak_kind,
                     "algo_bytes_per_launch": algo, "launch_ms": launch_ms,
                     "share_of_step": dom_ms / ms_step},
        "kernels": ktimes,
        "clocks": clk.summary(),
        "cpu_baseline": cpu,
        "reader": reader,
    }
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
