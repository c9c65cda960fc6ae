"""One (or a few) full censuses of a BASELINE config from device-resident
arrays (index build + both passes), for ncu captures and work counters.
Usage (GPU box): python profiles/census_once.py [config] [delta] [reps]
  config: powerlaw_50m_600m (default) | triadic_25m_100m | hubstress_100k_50m | powerlaw_1m_10m"""
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
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
if name in synth.GPU_CONFIGS:
    n, s, d, t = synth.GPU_CONFIGS[name]["fn"]()
else:
    n, s_, d_, t_ = synth.CONFIGS[name]["fn"]()
    s = torch.from_numpy(s_.view(np.int32)).cuda()
    d = torch.from_numpy(d_.view(np.int32)).cuda()
    t = torch.from_numpy(t_).cuda()
torch.cuda.synchronize()
for r in range(reps):
    t0 = time.time()
    census = tm.count_edges_device(n, s.numel(), s.data_ptr(), d.data_ptr(), t.data_ptr(), tm.RunConfig(delta=delta))
    print(json.dumps({"config": name, "delta": delta, "rep": r, "s": round(time.time() - t0, 4),
                      "census_total": int(np.asarray(census, np.uint64).sum())}), flush=True)
if os.environ.get("KTIMES"):  # per-kernel CUDA-event times of one more census
    tm.kernel_timing(enable=True, reset=True)
    tm.count_edges_device(n, s.numel(), s.data_ptr(), d.data_ptr(), t.data_ptr(), tm.RunConfig(delta=delta))
    torch.cuda.synchronize()
    tm.kernel_timing(enable=False)
    names = ["star_filter", "star_locate", "star_work", "tri_filter", "tri_wedge", "tri_long", "radix_upsweep", "radix_downsweep",
             "radix_scan", "scan", "gather_s", "s_offsets", "gather_p", "p_flags", "forward_scatter", "pack_edges", "pair_keys", "time_keys",
             "forward_off", "group_end", "pair_table", "tri_gate", "orient", "degree_class"]
    kt = {k: round(tm.kernel_time(k)[0], 3) for k in names if tm.kernel_time(k)[1]}
    print(json.dumps({"config": name, "delta": delta, "kernel_ms": kt}), flush=True)
ctx = tm.GraphContext.build_device(n, s.data_ptr(), d.data_ptr(), t.data_ptr(), s.numel())
tm.run_parallel(ctx, tm.RunConfig(delta=delta))
print(json.dumps({"config": name, "delta": delta, **ctx.run_stats()}), flush=True)
ctx.close()
