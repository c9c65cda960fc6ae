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
    rf = d["roofline"]
    rows.append((c["workload"], c.get("delta"), c.get("edges"), d["ms_per_step"], d["value"], d["e2e"]["value"],
                 rf["kernel"], rf["share_of_step"], rf["frac"], cpu.get("value"), d.get("census_total")))
print("| workload | δ | edges | ms/step | G edges/s (HBM-resident) | G edges/s e2e (host) | top kernel (share, HBM frac) "
      "| reference CPU M edges/s (16 thr, 2M-edge slice) | census total |")
print("|---|---|---|---|---|---|---|---|---|")
for r in rows:
    fr = f"{r[8]:.2f}" if r[8] is not None else "-"
    print(f"| {r[0]} | {r[1]} | {r[2]:,} | {r[3]:.2f} | {r[4]/1e9:.2f} | {r[5]/1e9:.2f} | {r[6]} ({100*r[7]:.0f} %, {fr}) | "
          f"{(r[9] or 0)/1e6:.2f} | {r[10]:,} |")
