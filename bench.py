"""bench.py -- exact 36-motif temporal census throughput on B200.

Step = one full census of the BASELINE workload from edge arrays resident in
HBM: GPU index build (radix sorts -> S / P / F layouts) + FAST-Star pass +
FAST-Tri pass + counter all-reduce (N > 1) + merge.  value = edges x steps /
max-over-ranks device time.  e2e = the same step through the C-ABI from
pinned HOST arrays, host->device copies and the counter read-back inside the
timed region.  Default workload: BASELINE config 4 (powerlaw_50m_600m, 50M
nodes / 600M edges, delta 3600 -- the middle of its delta sweep), the largest
single-GPU configuration.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config NAME] [--delta D] [--impl ours|reference]

--impl reference times the reference's own CPU implementation (oracle/_ref:
the unmodified reference sources; GraphContext::build + run_parallel with all
host threads) on a bounded time slice of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

MEASURED_PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")
METRIC = "temporal edges/sec, exact 36-motif count (1/2/4/8 B200); % of HBM roofline"
DEFAULT_CONFIG = "powerlaw_50m_600m"


# Algorithmic bytes per STEP for each kernel family:
# bytes that must cross HBM at least once.  Times are u32 offsets (narrow
# records) when the time span fits 32 bits, else int64 (wide).
#   radix_downsweep per key per digit pass: u64 key read + write, plus (narrow
#                 records) the u64 payload read + write
#                 node sort: 2m keys (node << 32 | record), ceil(nb/8) passes (the
#                 first reads the caller's src / dst / t, 8 B per record, when the
#                 input is time-ordered)
#                 pair sort: m keys (min << 32 | edge), ceil(nb/8) passes
#                 t sort:    m keys, ceil(tbits/8) passes (unsorted input only)
#   gather_s      (wide records only) per incident record: sorted key 8 + the
#                 16-byte edge record + S outputs t 8, nbr 4, ord 4, node 4; narrow
#                 records: the node sort's last pass writes S itself (same bytes as
#                 writing the sorted key + payload), then
#   s_offsets     per incident record: S node 4; per node: offset 4 written
#   gather_p      (wide records only) per edge: sorted key 8 + the 16-byte edge
#                 record + P outputs t 8, ord 4, min 4, max 4, w 4; narrow records:
#                 the pair sort's last pass writes P itself, then
#   p_flags       per edge: P min 4 + max 4 + w 4 read, w 4 written; per node pofs 4
#   pair_keys     per incident record: key 8 + S nbr 4 + S t 4; per edge the pair
#                 key 8 + payload 8 written
#   star_filter   per edge: P t 4 (8) + P w 4
#   tri_filter    per forward record (one per edge): F t 4 (8) + F node 4 + F nbr 4
#   scan          per mask word: 2 words read + 2 prefix words written
#   work kernels (random access; one 32-byte sector per dependent lookup):
#   star_locate   per candidate: list entry 4 + P record 16 + the S locate 32 + PS entry 8
#   star_work     per candidate: list entry 4 + P record 16 + its PS entry 8
#   tri_wedge     per short wedge: wedge 8 + two F records 24 + the closing lookup 32
#   tri_long      per long wedge: F record 12 + the closing lookup 32
def algo_bytes(n, m, t, stats=None):
    R = 2 * m
    nb = max(1, int(n - 1).bit_length())
    pbits = max(1, int(m - 1).bit_length())
    tb = int(int(t.max()) - int(t.min())).bit_length() if m else 0
    unsorted = bool(m > 1 and (np.diff(t) < 0).any())
    narrow = tb <= 32
    kv = 16 if narrow else 8  # key (+ payload) bytes per sorted element
    sort = R * kv * 2 * ((nb + 7) // 8)
    sort += m * kv * 2 * ((nb + 7) // 8)
    if unsorted:
        sort += m * (8 if tb + pbits <= 64 else 12) * 2 * ((tb + 7) // 8)
    elif narrow:
        sort -= R * 8  # the node sort's first pass reads the edge arrays (8 B per record), not packed records
    tw = 4 if narrow else 8
    eb = 8 if narrow else 16
    out = {"radix_downsweep": sort, "gather_s": R * (8 + eb + tw + 12), "gather_p": m * (8 + eb + tw + 16),
           "pair_keys": R * 16 + m * 16, "star_filter": m * (tw + 4), "tri_filter": m * (tw + 8),
           "scan": (R + m) // 32 * 16, "s_offsets": R * 4 + n * 4,
           "p_flags": m * 16 + n * 4}
    if stats:
        cand = stats["star_first_candidates"] + stats["star_third_candidates"]
        out["star_locate"] = cand * 60
        out["star_work"] = cand * 28
        out["tri_wedge"] = stats["short_wedges"] * 64
        out["tri_long"] = stats["long_wedges"] * 44
    return out


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def load_workload(name: str, delta=None):
    """(n, device arrays or None, host arrays, delta).  Configs 2-4 are
    generated on the GPU (configs 3/4 by the counter-based generators the
    reference's golden censuses were computed on) and kept there; the host
    copies feed the e2e leg and the CPU reference."""
    from paper_2204_09236_b200 import synth
    if name in synth.CONFIGS:
        cfg = synth.CONFIGS[name]
        n, src, dst, t = cfg["fn"]()
        return n, None, (src, dst, t), int(delta if delta is not None else cfg["delta"])
    cfg = synth.GPU_CONFIGS[name]
    n, src, dst, t = cfg["fn"]()
    d = delta if delta is not None else cfg["delta"]
    host = (src.cpu().numpy().view(np.uint32), dst.cpu().numpy().view(np.uint32), t.cpu().numpy())
    return n, (src, dst, t), host, int(d)


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


def reference_sample(src, dst, t, sample_edges):
    """The earliest `sample_edges` edges in time order (ingestion order kept),
    node ids relabelled densely: a time slice of the workload as a graph of
    its own (the reference then sizes its per-node tables to the slice)."""
    if np.all(t[1:] >= t[:-1]):
        order = np.arange(min(sample_edges, len(t)))
    else:
        order = np.sort(np.argsort(t, kind="stable")[:sample_edges])
    s, d, tt = src[order], dst[order], t[order]
    ids, inv = np.unique(np.concatenate([s, d]), return_inverse=True)
    return len(ids), inv[:len(s)].astype(np.uint32), inv[len(s):].astype(np.uint32), tt


def cpu_reference(sample, delta, steps, warmup, threads):
    """Time the reference's own pipeline on a sample: TemporalGraph::build +
    GraphContext::build + run_parallel (graph.cpp:13-44, executor.cpp:149-215),
    wall time of those calls only (the shim's node-id strings and edge
    vector are filled before the clock starts)."""
    from oracle import Reference
    R = Reference()
    n, s, d, tt = sample
    times = []
    census = None
    for i in range(warmup + steps):
        census, mb, mc = R.pipeline(n, s, d, tt, delta, threads)
        if i >= warmup:
            times.append((mb + mc) * 1e-3)
    sec = float(np.mean(times))
    return {"value": len(s) / sec, "sec_per_step": sec, "edges": int(len(s)), "census_total": int(census.sum())}


def h2d_peak_gbps(dev):
    """Pinned host -> device copy bandwidth (1 GiB, best of 3): the link the
    e2e leg's input copies run on."""
    import torch
    h = torch.empty(1 << 30, dtype=torch.uint8).pin_memory()
    d = torch.empty(1 << 30, dtype=torch.uint8, device=dev)
    best = 0.0
    for _ in range(3):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        d.copy_(h, non_blocking=True)
        e1.record()
        torch.cuda.synchronize()
        best = max(best, (1 << 30) / (e0.elapsed_time(e1) * 1e-3) / 1e9)
    del h, d
    return best


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default=DEFAULT_CONFIG)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--reader", action="store_true", help="also time the GPU edge-list reader (config 1 sizes)")
    ap.add_argument("--no-reader", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--cpu-sample-edges", type=int, default=2_000_000)
    ap.add_argument("--delta", type=int, default=None, help="override the config's delta")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="counter all-reduce backend (gloo: CPU tensors, for multi-rank tests on one GPU)")
    ap.add_argument("--partition", default="time", choices=["time", "centers"],
                    help="N>1: time slices of the first edge (each rank indexes only its slice) or "
                         "center ranges over a replicated graph")
    ap.add_argument("--same-device", action="store_true",
                    help="testing only: every rank uses cuda:0 (independent kernels, gloo reduce)")
    ap.add_argument("--force-dist", action="store_true",
                    help="testing only: take the N>1 path (process group, counter all-reduce) at world size 1, "
                         "so the NCCL reduce runs on a single-GPU box")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    threads = os.cpu_count() or 1

    if args.impl == "reference":
        if rank != 0:
            return
        n, m, (src, dst, t), delta = load_workload_host(args.config, args.delta, args.cpu_sample_edges)
        sample = reference_sample(src, dst, t, min(args.cpu_sample_edges, m))
        del src, dst, t
        res = cpu_reference(sample, delta, args.steps, args.warmup, threads)
        desc = (f"earliest {res['edges']} of {m} edges in time order, node ids relabelled densely "
                f"({sample[0]} nodes); wall time of TemporalGraph::build + GraphContext::build + run_parallel "
                f"({threads} std::threads)")
        line = {"metric": METRIC, "value": res["value"], "unit": "edges/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": res["sec_per_step"] * 1e3, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "int64", "data": "synthetic",
                "impl": "reference",
                "config": {"workload": args.config, "nodes": int(n), "edges": int(m), "delta": int(delta),
                           "parallelism": "cpu", "sample": desc},
                "cpu_baseline": {"value": res["value"], "unit": "edges/s", "cores": threads, "kind": "reference",
                                 "sample": desc},
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
    multi = world > 1 or (args.force_dist and "RANK" in os.environ)
    if multi:
        import torch.distributed as dist
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")
    import paper_2204_09236_b200 as tm

    n, dev_arrays, (src, dst, t), delta = load_workload(args.config, args.delta)
    m = len(src)
    tb = int(int(t.max()) - int(t.min())).bit_length() if m else 0
    base_cfg = {"workload": args.config, "nodes": int(n), "edges": int(m), "delta": int(delta),
                "inputs": ("synthetic edge list (seed 2204), "
                           + ("ingestion order = time order" if m < 2 or bool(np.all(t[1:] >= t[:-1]))
                              else "not time-ordered (the GPU time sort runs)")),
                "l2": "inputs + indexes exceed the 126 MB L2 many times over; no explicit flush"}

    stream = torch.cuda.Stream(device=dev)
    sptr = stream.cuda_stream
    cfg = tm.RunConfig(delta=delta)
    center = (0, 0)
    if world > 1 and args.partition == "time":
        # each rank holds the edges with t in [lo, hi + delta) and owns the
        # instances whose earliest edge has t in [lo, hi): exact partition
        from paper_2204_09236_b200.distributed import time_slice_bounds, time_slice_mask
        lo, hi = time_slice_bounds(t, world, delta)[rank]  # balanced by estimated work
        keep = time_slice_mask(t, lo, hi, delta)
        src, dst, t = src[keep], dst[keep], t[keep]
        dev_arrays = None
        cfg = tm.RunConfig(delta=delta, first_edge_t_end=hi)
    m_local = len(src)
    if dev_arrays is None:
        d_src = torch.from_numpy(src.view(np.int32)).to(dev)
        d_dst = torch.from_numpy(dst.view(np.int32)).to(dev)
        d_t = torch.from_numpy(t).to(dev)
    else:
        d_src, d_dst, d_t = dev_arrays
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
    # work counters of this workload (for the work kernels' byte models)
    ctx = tm.GraphContext.build_device(n, d_src.data_ptr(), d_dst.data_ptr(), d_t.data_ptr(), m_local, stream=sptr)
    tm.run_parallel(ctx, cfg)
    stats = ctx.run_stats()
    ctx.close()
    del ctx
    torch.cuda.synchronize()
    torch.cuda.empty_cache()

    raw = np.zeros(56, np.uint64)
    from paper_2204_09236_b200.distributed import allreduce_counters

    def reduce_raw(census):
        if multi:  # one all-reduce of the 56 counters, exact (32-bit halves), checked on merge
            with torch.cuda.stream(stream):
                tot = allreduce_counters(raw, device=red_dev)
            census = tm.merge_census(tm.StarCounter(tot[:24]), tm.PairCounter(tot[24:32]), tm.TriCounter(tot[32:]),
                                     cfg.triangle_mode).counts
        return census

    def step(host: bool):
        if host:
            census = tm.count_edges(n, h_src.numpy().view(np.uint32), h_dst.numpy().view(np.uint32), h_t.numpy(),
                                    cfg, stream=sptr, raw_out=raw, center=center)
        else:
            census = tm.count_edges_device(n, m_local, d_src.data_ptr(), d_dst.data_ptr(), d_t.data_ptr(), cfg,
                                           stream=sptr, center=center, raw_out=raw)
        return reduce_raw(census)

    def device_ms(fn, steps, warmup):
        for _ in range(warmup):
            census = fn()
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        l0 = tm.kernel_launches()
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            ev0.record(stream)
        census = fn(steps)
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

    def loop(host):
        def run(k=1):
            for _ in range(k):
                census = step(host)
            return census
        return run

    def pipelined(k=1):
        """e2e through tm_count_edges_async: batch i+1's host->device copy
        overlaps batch i's census (two batches staged); every step still
        copies its inputs from pinned host memory and reads its counters back."""
        from collections import deque

        def submit():
            return tm.count_edges_async(n, h_src.numpy().view(np.uint32), h_dst.numpy().view(np.uint32),
                                        h_t.numpy(), cfg, stream=sptr)

        q = deque()
        census = None
        for _ in range(k):
            q.append(submit())
            if len(q) > 1:
                census = reduce_raw(q.popleft().result(raw_out=raw))
        while q:
            census = reduce_raw(q.popleft().result(raw_out=raw))
        return census

    with ClockSampler(local) as clk:
        ms_step, census, launches = device_ms(loop(False), args.steps, args.warmup)
    ms_e2e_sync, census_e2e, _ = device_ms(loop(True), max(2, args.steps // 2), args.warmup)
    assert (census == census_e2e).all(), "device and host paths disagree"
    e2e_api = "tm_count_edges_async (two batches in flight: copy of batch i+1 overlaps census i)"
    h2d_bytes = int(m_local * 16)
    if tuple(center) == (0, 0):
        # >= 4 batches: the pipeline fill (first copy, last census) is amortised;
        # two warm-up batches touch both staging slots
        ms_e2e, census_pipe, _ = device_ms(pipelined, max(4, args.steps), 2)
        assert (census == census_pipe).all(), "device and pipelined host paths disagree"
        h2d_bytes = tm.async_h2d_bytes()
        if h2d_bytes < m_local * 16:
            per_edge = h2d_bytes // max(1, m_local)
            e2e_api += (f"; timestamps travel as per-block i64 bases + u{(per_edge - 8) * 8} offsets packed by host "
                        f"worker threads inside the timed region ({per_edge} B per edge on the link)")
    else:  # center ranges go through the synchronous API only
        ms_e2e = ms_e2e_sync
        e2e_api = "tm_count_edges (one batch at a time)"
    h2d = h2d_peak_gbps(dev)

    # per-kernel device time with CUDA events on the launching stream (separate instrumented pass)
    tm.kernel_timing(enable=True, reset=True)
    kk = max(2, min(args.steps, 3))
    for _ in range(kk):
        step(False)
    torch.cuda.synchronize()
    tm.kernel_timing(enable=False)
    names = ["star_filter", "star_locate", "star_work", "tri_filter", "tri_wedge", "tri_long", "radix_upsweep",
             "radix_downsweep", "radix_scan", "scan", "gather_s", "s_offsets", "gather_p", "p_flags", "forward_scatter", "pack_edges",
             "pair_keys", "time_keys", "perm_from_keys", "validate", "offsets", "forward_off", "group_end",
             "pair_table", "tri_gate", "orient", "degree_class"]
    ktimes = {}
    for nm in names:
        tot_ms, cnt = tm.kernel_time(nm)
        if cnt:
            ktimes[nm] = {"ms_per_step": tot_ms / kk, "launches_per_step": cnt / kk}
    abytes = algo_bytes(n, m_local, t, stats)
    for k, v in ktimes.items():
        if k in abytes:
            v["algo_GBps"] = abytes[k] / (v["ms_per_step"] * 1e-3) / 1e9
    # the roofline kernel: the one with the most device time per step
    dom = max(ktimes, key=lambda k: ktimes[k]["ms_per_step"])
    dom_ms = ktimes[dom]["ms_per_step"]
    dom_launches = max(1.0, ktimes[dom]["launches_per_step"])
    launch_ms = dom_ms / dom_launches
    peak, peak_kind = peaks()
    algo = abytes.get(dom, 0) / dom_launches
    achieved = algo / (launch_ms * 1e-3) / 1e9 if algo else None
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "r02", f"traffic_{dom}_{args.config}_{delta}.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get("bytes_per_launch")
        except Exception:
            traffic = None

    reader = None
    if world == 1 and args.reader:
        reader = time_reader(tm, torch, dev, stream, sptr, m_local, d_src, d_dst, d_t, cfg, census)

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
                sample = reference_sample(src, dst, t, min(args.cpu_sample_edges, m))
                res = cpu_reference(sample, delta, 1, 0, threads)
                cpu = {"value": res["value"], "unit": "edges/s", "cores": threads, "kind": "reference",
                       "sample": f"earliest {res['edges']} of {m} edges in time order, node ids relabelled "
                                 f"({sample[0]} nodes); one run of TemporalGraph::build + GraphContext::build + "
                                 f"run_parallel with {threads} std::threads"}
        except Exception as ex:  # pragma: no cover
            log("cpu baseline failed:", ex)

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
        "census": [int(x) for x in census],
        "e2e": {"value": m / (ms_e2e * 1e-3), "unit": "edges/s", "h2d_bytes_per_step": h2d_bytes,
                "d2h_bytes_per_step": int(56 * 8 + 36 * 8), "ms_per_step": ms_e2e,
                "api": e2e_api, "h2d_GBps_measured": h2d,
                "h2d_bound_ms": h2d_bytes / (h2d * 1e9) * 1e3,
                "sync_api": {"value": m / (ms_e2e_sync * 1e-3), "ms_per_step": ms_e2e_sync,
                             "api": "tm_count_edges (one batch at a time)"}},
        "gpu_launches": int(launches),
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak if achieved else None, "traffic": traffic, "peak_kind": peak_kind,
                     "algo_bytes_per_launch": algo, "launch_ms": launch_ms,
                     "share_of_step": dom_ms / ms_step},
        "kernels": ktimes,
        "work": stats,
        "clocks": clk.summary(),
        "cpu_baseline": cpu,
    }
    if reader is not None:
        line["reader"] = reader
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def load_workload_host(name, delta=None, prefix=None):
    """(n, m, host arrays, delta) for the reference arm, generated on the host
    (numpy twins of the GPU generators).  Config 4 is time-ordered, so only
    its first `prefix` edges are generated."""
    from paper_2204_09236_b200 import synth
    if name in synth.CONFIGS:
        n, _, (s, dd, t), d = load_workload(name, delta)
        return n, len(s), (s, dd, t), d
    cfg = synth.GPU_CONFIGS[name]
    d = int(delta if delta is not None else cfg["delta"])
    if name == "powerlaw_50m_600m":
        n, s, dd, t = synth.power_law_hashed(lo=0, hi=prefix)
        return n, 600_000_000, (s, dd, t), d
    if name == "triadic_25m_100m":
        n, s, dd, t = synth.triadic_hashed()
        return n, len(s), (s, dd, t), d
    n, s, dd, t = synth.hub_stress()
    return n, len(s), (s, dd, t), d


def time_reader(tm, torch, dev, stream, sptr, m_local, d_src, d_dst, d_t, cfg, census):
    """The edge-list reader in front of the path: the same edges as "SRC DST T"
    text, parsed on the GPU from device memory and from host memory; the
    parsed arrays are counted once and must give the same census."""
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
    return {"what": "tm_parse_edge_list: the reference's parse_edge_list (graph.cpp:73) on the GPU",
            "text_bytes": int(nbytes), "lines": int(m_local),
            "device_text": {"ms": ms_dev, "GB_per_s": nbytes / (ms_dev * 1e-3) / 1e9,
                            "lines_per_s": m_local / (ms_dev * 1e-3)},
            "host_text": {"ms": ms_host, "GB_per_s": nbytes / (ms_host * 1e-3) / 1e9,
                          "lines_per_s": m_local / (ms_host * 1e-3)}}


if __name__ == "__main__":
    main()
