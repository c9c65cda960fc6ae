"""Config 4 (600M edges) at delta 86400 once: the wedge-bound triangle case,
for an ncu capture of tri_long / tri_wedge.  Usage (GPU box):
  python profiles/config4_tri.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2204_09236_b200 as tm  # noqa: E402
from paper_2204_09236_b200 import synth  # noqa: E402

n, s, d, t = synth.power_law_hashed(device="cuda")
torch.cuda.synchronize()
ctx = tm.GraphContext.build_device(n, s.data_ptr(), d.data_ptr(), t.data_ptr(), s.numel())
t0 = time.time()
census = tm.run_parallel(ctx, tm.RunConfig(delta=86400, motifs=tm.MotifFilter(star=False, pair=False)))
print("count_s", round(time.time() - t0, 3), "total", census.total(), ctx.run_stats(), flush=True)
ctx.close()
