#!/bin/bash
# Copy a gpurun_out/r02cap/ capture (profiles/capture_r02.sh: config 4,
# powerlaw_50m_600m, 600M edges, delta 3600) into profiles/r02/.
set -e
cd "$(dirname "$0")/.."
G=gpurun_out/r02cap; P=profiles/r02
mkdir -p $P
rm -f $P/ncu_*.txt $P/lines_*.txt $P/traffic_*.json
cp $G/ncu_*.txt $G/lines_*.txt $G/traffic_*.json $G/launches.txt $G/launches.csv $G/census_once.jsonl $P/
cp $G/bench.json $P/bench.json
