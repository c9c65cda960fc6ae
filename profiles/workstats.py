"""Print the GPU path's work counters (star candidates, wedges) per config/delta.
Usage (GPU box): python profiles/workstats.py"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2204_09236_b200 as tm  # noqa: E402
from paper_2204_09236_b200 import synth  # noqa: E402


def run(name, n, src, dst, t, deltas):
    if not torch.is_tensor(src):
        src = torch.from_numpy(src.view("int32")).cuda()
        dst = torch.from_numpy(dst.view("int32")).cuda()
        t = torch.from_numpy(t).cuda()
    torch.cuda.synchronize()
    ctx = tm.GraphContext.build_device(n, src.data_ptr(), dst.data_ptr(), t.data_ptr(), src.numel())
    for d in deltas:
        t0 = time.time()
        census = tm.run_parallel(ctx, tm.RunConfig(delta=d))
        dt = time.time() - t0
        print(json.dumps({"config": name, "delta": d, "edges": int(src.numel()), "census_total": census.total(),
                          "count_s": round(dt, 4), **ctx.run_stats()}), flush=True)
    ctx.close()


if __name__ == "__main__":
    run("powerlaw_1m_10m", *synth.power_law(), [600, 3600, 86400])
    run("hubstress_100k_50m", *synth.hub_stress_gpu(), [600, 3600])
    run("triadic_25m_100m", *synth.triadic_hashed(device="cuda"), [3600, 86400])
    run("powerlaw_50m_600m", *synth.power_law_hashed(device="cuda"), [600, 3600, 86400])
