#!/bin/bash
# GPU-box call: the reference's run_parallel on the WHOLE config 4 (600M edges)
# on the host cores in the background (tests/golden/config4_full_reference.json),
# kernel A/B runs on the GPU meanwhile.   profiles/call_golden4.sh <deltas> <kab libs...>
out=gpurun_out/g4; mkdir -p $out
D=${1:-600,3600}; shift
(GOLDEN_OUT=$out GOLDEN_DELTAS=$D timeout 4000 python tests/golden/make_golden.py --only-extra --config4-full \
   > $out/golden.log 2>&1; echo "golden rc $?" >> $out/golden.log) &
GP=$!
sleep 60
if [ $# -gt 0 ]; then
  bash profiles/kab.sh 2 powerlaw_50m_600m 3600 "$@" > $out/kab3600.jsonl 2> $out/kab.err
  bash profiles/kab.sh 1 powerlaw_50m_600m 86400 "$@" > $out/kab86400.jsonl 2>> $out/kab.err
fi
free -g > $out/free.txt
wait $GP
tail -5 $out/golden.log
