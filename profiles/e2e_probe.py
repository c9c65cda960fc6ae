"""Host-side timeline of the pipelined e2e API (tm_count_edges_async /
wait) on a config: wall time of every submit / result call, to see whether
batch i+1's host->device copy overlaps batch i's census.
Usage (GPU box): python profiles/e2e_probe.py [config] [delta] [batches]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2204_09236_b200 as tm  # noqa: E402
from paper_2204_09236_b200 import synth  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "powerlaw_50m_600m"
delta = int(sys.argv[2]) if len(sys.argv) > 2 else 3600
nb = int(sys.argv[3]) if len(sys.argv) > 3 else 6
if name in synth.GPU_CONFIGS:
    n, s, d, t = synth.GPU_CONFIGS[name]["fn"]()
    hs, hd, ht = s.cpu().pin_memory(), d.cpu().pin_memory(), t.cpu().pin_memory()
    del s, d, t
else:
    n, s_, d_, t_ = synth.CONFIGS[name]["fn"]()
    hs = torch.from_numpy(s_.view(np.int32)).pin_memory()
    hd = torch.from_numpy(d_.view(np.int32)).pin_memory()
    ht = torch.from_numpy(t_).pin_memory()
torch.cuda.empty_cache()
cfg = tm.RunConfig(delta=delta)
st = torch.cuda.Stream()
args = (hs.numpy().view(np.uint32), hd.numpy().view(np.uint32), ht.numpy())
T0 = time.perf_counter()
log = []


def mark(what):
    log.append((what, round((time.perf_counter() - T0) * 1e3, 2)))


q = []
for b in range(nb):
    mark(f"submit {b} start")
    q.append(tm.count_edges_async(n, *args, cfg, stream=st.cuda_stream))
    mark(f"submit {b} end")
    if len(q) > 1:
        q.pop(0).result()
        mark(f"result {b - 1}")
while q:
    q.pop(0).result()
    mark("result last")
torch.cuda.synchronize()
print(json.dumps({"config": name, "delta": delta, "timeline_ms": log}), flush=True)
t1 = time.perf_counter()
for b in range(3):
    tm.count_edges(n, *args, cfg, stream=st.cuda_stream)
print(json.dumps({"sync_ms_per_batch": round((time.perf_counter() - t1) * 1e3 / 3, 2)}), flush=True)
