"""Per-step fixed overhead: wall time and phase timings of count_edges_device at
small edge counts (usage on the GPU box: python profiles/overhead.py)."""
import sys, os, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2204_09236_b200 as tm
from paper_2204_09236_b200 import synth
for m in (1000, 200000, 2000000):
    n, s, d, t = synth.uniform(10000, m, 10**6 - 1, 2204)
    ds = torch.from_numpy(s.view(np.int32)).cuda(); dd = torch.from_numpy(d.view(np.int32)).cuda(); dt = torch.from_numpy(t).cuda()
    st = torch.cuda.Stream()
    cfg = tm.RunConfig(delta=1000)
    for rep in range(3):
        tmg = tm.PhaseTimings() if hasattr(tm, 'PhaseTimings') else None
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(10):
            tm.count_edges_device(n, m, ds.data_ptr(), dd.data_ptr(), dt.data_ptr(), cfg, stream=st.cuda_stream, timings=tmg)
        torch.cuda.synchronize()
        dtm = (time.perf_counter() - t0) / 10
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(10):
        tm.count_edges_device(n, m, ds.data_ptr(), dd.data_ptr(), dt.data_ptr(), cfg, stream=st.cuda_stream)
    torch.cuda.synchronize()
    dtn = (time.perf_counter() - t0) / 10
    print(m, "wall ms/step", round(dtm * 1e3, 3), "no-timings", round(dtn * 1e3, 3), "phases", tmg.index_ms if tmg else None, tmg.star_pair_ms if tmg else None, tmg.triangle_ms if tmg else None, tmg.merge_ms if tmg else None, flush=True)
