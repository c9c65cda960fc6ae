#!/bin/bash
# Session-4 first call: bench at HEAD (quiet box), per-kernel times at both
# deltas, then the whole-config-4 reference golden on the host cores while the
# GPU suite runs.
set -x
out=gpurun_out/s4; mkdir -p $out
nproc > $out/host.txt; free -g >> $out/host.txt
python bench.py > $out/bench.json 2> $out/bench.err; echo bench=$?
for d in 3600 86400; do KTIMES=1 timeout 600 python profiles/census_once.py powerlaw_50m_600m $d 2; done > $out/c4.jsonl 2> $out/c4.err
(GOLDEN_OUT=$out GOLDEN_DELTAS=${1:-600} timeout 2700 python tests/golden/make_golden.py --only-extra --config4-full \
   > $out/golden.log 2>&1; echo "golden rc $?" >> $out/golden.log) &
GP=$!
timeout 2400 python -m pytest tests -m gpu -q -x > $out/gputest.log 2>&1; echo "pytest rc $?" >> $out/gputest.log
tail -3 $out/gputest.log
free -g >> $out/host.txt
wait $GP
tail -5 $out/golden.log
