"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV) into
per-kernel totals and shares.  Usage: python summarize_launches.py launches.csv"""
import csv
import re
import sys
from collections import defaultdict

rows = list(csv.DictReader(l for l in open(sys.argv[1]) if l.startswith('"')))
tot = defaultdict(float)
cnt = defaultdict(int)
for r in rows:
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = r["Kernel Name"]
    m = re.search(r"(\w+_kernel|radix_\w+|scan_\w+)", name)
    key = m.group(1) if m else name[:40]
    if "radix_downsweep" in name or "radix_upsweep" in name:
        key += "<u64>" if "unsigned long" in name.split("(")[1] else "<u32>"
    tot[key] += float(r["Metric Value"])
    cnt[key] += 1
all_ns = sum(tot.values())
print(f"{'kernel':40s} {'launches':>8s} {'total_us':>10s} {'avg_us':>9s} {'share':>6s}")
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{k:40s} {cnt[k]:8d} {v/1e3:10.1f} {v/1e3/cnt[k]:9.1f} {100*v/all_ns:5.1f}%")
print(f"{'TOTAL':40s} {sum(cnt.values()):8d} {all_ns/1e3:10.1f}")
