"""Config 1 (1M nodes / 10M edges) counted once at delta 86400 -- the
wedge-heavy regime where tri_long / star_work dominate -- for ncu captures.
Usage (GPU box): python profiles/bigdelta_profile.py [delta]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2204_09236_b200 as tm  # noqa: E402
from paper_2204_09236_b200 import synth  # noqa: E402

delta = int(sys.argv[1]) if len(sys.argv) > 1 else 86400
n, s, d, t = synth.CONFIGS["powerlaw_1m_10m"]["fn"]()
ds = torch.from_numpy(s.view(np.int32)).cuda()
dd = torch.from_numpy(d.view(np.int32)).cuda()
dt = torch.from_numpy(t).cuda()
ctx = tm.GraphContext.build_device(n, ds.data_ptr(), dd.data_ptr(), dt.data_ptr(), len(s))
census = tm.run_parallel(ctx, tm.RunConfig(delta=delta))
print("total", census.total(), ctx.run_stats(), flush=True)
ctx.close()
