"""Per-source-line stall samples and executed instructions of one kernel from
an ncu report: python profiles/ncu_lines.py report.ncu-rep [kernel-substring] [min%]
(uses `ncu --page source --print-source cuda,sass`)."""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
want = sys.argv[2] if len(sys.argv) > 2 else ""
thr = float(sys.argv[3]) if len(sys.argv) > 3 else 0.5
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
agg = collections.defaultdict(lambda: [0, 0])
src = {}
fn = path = None
seen = set()
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        path = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        fn = r[1]
        continue
    if r[0] == "Line No" or not r[0].isdigit() or want not in (fn or ""):
        continue
    key = (fn, path, int(r[0]))
    if key in seen:  # a function's listing repeats per file; count each line once
        continue
    seen.add(key)
    try:
        s, e = int(r[4]), int(r[7])
    except ValueError:
        continue
    a = agg[(path, int(r[0]))]
    a[0] += s
    a[1] += e
    src[(path, int(r[0]))] = r[1]
ts = sum(v[0] for v in agg.values()) or 1
te = sum(v[1] for v in agg.values()) or 1
print(f"stall samples {ts}, warp instructions {te}")
for k, (s, e) in sorted(agg.items()):
    if 100 * s / ts >= thr or 100 * e / te >= thr:
        print(f"{k[0][:18]:18s}:{k[1]:<4d} {100*s/ts:5.1f}% stall {100*e/te:5.1f}% inst  {src[k][:90]}")
