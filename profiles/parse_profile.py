"""The config-1 edge list as text on the device, parsed three times by
tm_parse_edge_list -- for an ncu launch list / capture of the reader kernels.
Usage (GPU box): python profiles/parse_profile.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2204_09236_b200 as tm  # noqa: E402
from paper_2204_09236_b200 import synth  # noqa: E402

n, s, d, t = synth.CONFIGS["powerlaw_1m_10m"]["fn"]()
ds = torch.from_numpy(s.view(np.int32)).cuda()
dd = torch.from_numpy(d.view(np.int32)).cuda()
dt = torch.from_numpy(t).cuda()
m = len(s)
nb = tm.write_edge_list_device(m, ds.data_ptr(), dd.data_ptr(), dt.data_ptr())
text = torch.empty(nb + 16, dtype=torch.uint8, device="cuda")
tm.write_edge_list_device(m, ds.data_ptr(), dd.data_ptr(), dt.data_ptr(), text.data_ptr())
torch.cuda.synchronize()
for _ in range(3):
    el = tm.parse_edge_list_gpu((text.data_ptr(), nb))
    print("parsed", el.n, el.m, flush=True)
    el.close()
