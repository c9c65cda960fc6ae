"""Reproducibility check for the GPU config generators and the counting path:
hashes the generated config-4 input and counts it three times.  Two runs of
this script must print identical lines.  Usage (GPU box): python profiles/det_check.py"""
import sys, os, json, hashlib
sys.path.insert(0, os.getcwd())
import torch, numpy as np
import paper_2204_09236_b200 as tm
from paper_2204_09236_b200 import synth
n, src, dst, t = synth.power_law_hashed(device="cuda")
torch.cuda.synchronize()
h = hashlib.sha1()
for a in (src, dst, t):
    h.update(a.view(torch.uint8)[::9973].cpu().numpy().tobytes())
    h.update(str(int(a.long().sum().item()) if a.dtype != torch.int64 else int((a % 1000003).sum().item())).encode())
print("input hash", h.hexdigest(), flush=True)
for rep in range(3):
    ctx = tm.GraphContext.build_device(n, src.data_ptr(), dst.data_ptr(), t.data_ptr(), src.numel())
    for d in (600,):
        raw, _ = tm.run_parallel_raw(ctx, tm.RunConfig(delta=d), 0, n)
        a = raw.as_array()
        print(rep, d, "star", int(a[:24].sum()), "pair", int(a[24:32].sum()), "tri", int(a[32:].sum()), flush=True)
    ctx.close()
