"""CPU, world_size 2 over gloo: the multi-GPU host path (degree-cost center
partition -> per-rank counters -> one all-reduce -> merge) reproduces the
single-process census.  Per-rank compute here is the oracle's per-center
counters (test stand-in for the GPU kernels), so this checks the partition
and reduction logic, not the kernels."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_q, n, src, dst, t, delta):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import Oracle
    from paper_2204_09236_b200.distributed import allreduce_counters, partition_bounds
    O = Oracle()
    g = O.build_graph(n, src, dst, t)
    deg = np.array([O.degree(g, u) for u in range(n)], np.uint64)
    cost = np.concatenate([[0], np.cumsum(deg)]).astype(np.uint64)
    b, e = partition_bounds(cost, world)[rank]
    raw = np.zeros(56, np.uint64)
    for u in range(b, e):
        s = int(deg[u])
        st, pr = O.star_pair_at_center(g, u, delta, 0, max(s - 2, 0))
        tr = O.triangles_at_center(g, u, delta, 0, max(s - 1, 0))
        raw[:24] += st; raw[24:32] += pr; raw[32:] += tr
    tot = allreduce_counters(raw)
    census = O.merge_census(tot[:24], tot[24:32], tot[32:])
    out_q.put((rank, (b, e), census.tolist()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4, 8])
def test_gloo_partition_allreduce_matches_single(world, oracle):
    n, m, delta = 60, 2500, 150
    src, dst, t = oracle.generate_random_graph(n, m, 8000, 4242)
    g = oracle.build_graph(n, src, dst, t)
    expect = oracle.census(g, delta).tolist()
    assert sum(expect) > 0 and sum(1 for x in expect if x) > 30
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, n, src, dst, t, delta)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    assert res[0][1][0] == 0 and res[-1][1][1] == n
    assert all(a[1][1] == b[1][0] for a, b in zip(res, res[1:]))
    for _, _, census in res:
        assert census == expect


def _slice_worker(rank, world, port, out_q, n, src, dst, t, delta):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import Oracle
    from paper_2204_09236_b200.distributed import allreduce_counters, time_slice_bounds, time_slice_mask
    O = Oracle()
    lo, hi = time_slice_bounds(t, world, delta)[rank]
    keep = time_slice_mask(t, lo, hi, delta)
    g = O.build_graph(n, src[keep], dst[keep], t[keep])
    part = O.census_bruteforce_before(g, delta, hi if hi is not None else 2 ** 63 - 1)
    tot = allreduce_counters(part)
    out_q.put((rank, (lo, hi), int(keep.sum()), tot.tolist()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3, 4, 8])
def test_gloo_time_slices_match_single(world, oracle):
    """Time-slice partition logic on CPU: each rank keeps t in [lo, hi + delta),
    counts instances whose earliest edge has t < hi (bounds balanced by the
    estimated work), one exact all-reduce."""
    n, m, delta = 30, 1500, 40
    src, dst, t = oracle.generate_random_graph(n, m, 2000, 777)
    g = oracle.build_graph(n, src, dst, t)
    expect = oracle.census_bruteforce(g, delta).tolist()
    assert sum(expect) > 0 and sum(1 for x in expect if x) > 30
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_slice_worker, args=(r, world, port, q, n, src, dst, t, delta))
             for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert sum(r[2] for r in res) < m + world * m // 10  # overlap is only the delta margins
    assert res[0][1][0] is None and res[-1][1][1] is None
    for r in res:
        assert r[3] == expect


def _overflow_worker(rank, world, port, out_q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2204_09236_b200.distributed import allreduce_counters
    from paper_2204_09236_b200.tmotif import CounterOverflowError
    raw = np.zeros(56, np.uint64)
    raw[5] = np.uint64(2 ** 63 + 7)  # every rank: 2^63 + 7 -> the total wraps a u64
    raw[6] = np.uint64(2 ** 62)      # 2 * 2^62 = 2^63: fits
    try:
        allreduce_counters(raw)
        out_q.put((rank, "no error"))
    except CounterOverflowError:
        out_q.put((rank, "overflow"))
    raw[5] = 0
    tot = allreduce_counters(raw)
    out_q.put((rank, int(tot[6])))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_allreduce_is_exact_and_checked():
    """The cross-rank merge raises CounterOverflowError when a total passes
    2^64 - 1 (the reference's checked partial merge, executor.cpp:173-179)
    and is exact below it."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_overflow_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(2 * world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert sorted(v for _, v in res if isinstance(v, str)) == ["overflow", "overflow"]
    assert [v for _, v in res if not isinstance(v, str)] == [2 ** 63, 2 ** 63]
