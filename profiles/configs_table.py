"""Markdown table of a profiles/configs_sweep.sh run."""
import glob
import json
import os
import sys

rows = []
for p in sorted(glob.glob(os.path.join(sys.argv[1], "*.json"))):
    try:
        d = json.load(open(p))
    except Exception:
        continue
    c = d["config"]
    cpu = d.get("cpu_baseline") or {}
    rows.append((c["workload"], c.get("delta"), c.get("edges"), d["ms_per_step"], d["value"], d["e2e"]["value"],
                 d["roofline"]["frac"], cpu.get("value"), d.get("census_total")))
print("| workload | δ | edges | ms/step | G edges/s (HBM-resident) | G edges/s e2e (host) | downsweep HBM frac | reference CPU M edges/s (16 thr, 1M-edge slice) | census total |")
print("|---|---|---|---|---|---|---|---|---|")
for r in rows:
    print(f"| {r[0]} | {r[1]} | {r[2]:,} | {r[3]:.2f} | {r[4]/1e9:.2f} | {r[5]/1e9:.2f} | {r[6]:.2f} | "
          f"{(r[7] or 0)/1e6:.2f} | {r[8]:,} |")
