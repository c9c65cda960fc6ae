"""Summarise a sortbench variant sweep log (lines '== <binary>' followed by
sortbench output): min downsweep ms per sort and stability check per variant."""
import collections
import re
import sys

d = collections.defaultdict(list)
bad = collections.Counter()
cur = key = None
for line in open(sys.argv[1]):
    if line.startswith("=="):
        cur = line.split("/")[-1].strip()
        continue
    m = re.match(r"(node|pair) keys.*best ([\d.]+) ms.*unstable=(\d+)", line)
    if m:
        key = m.group(1)
        d[(cur, key, "best")].append(float(m.group(2)))
        bad[cur] += int(m.group(3))
    m = re.match(r"\s+radix_downsweep\s+([\d.]+)", line)
    if m:
        d[(cur, key, "down")].append(float(m.group(1)))
for v in sorted({k[0] for k in d}):
    print(f"{v:14s} node down {min(d[(v,'node','down')]):.4f}  pair down {min(d[(v,'pair','down')]):.4f}  "
          f"node sort {min(d[(v,'node','best')]):.3f}  pair sort {min(d[(v,'pair','best')]):.3f}  unstable {bad[v]}")
