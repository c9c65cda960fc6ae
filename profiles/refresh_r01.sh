#!/bin/bash
# Rebuild profiles/r01/ from a gpurun_out/r01/ capture (bench.json,
# launches.csv, full2.ncu-rep, workstats.jsonl) made by the commands in
# profiles/r01/README.md.
set -e
cd "$(dirname "$0")/.."
G=gpurun_out/r01; P=profiles/r01; R=$G/full2.ncu-rep
rm -f $P/ncu_*.txt $P/traffic_*.json
python profiles/ncu_summary.py $R --kernel radix_downsweep --index 0 --algo 320000000 > $P/ncu_radix_downsweep_node_pass1.txt
python profiles/ncu_summary.py $R --kernel radix_downsweep --index 2 --algo 320000000 > $P/ncu_radix_downsweep_node_pass3.txt
python profiles/ncu_summary.py $R --kernel radix_downsweep --index 3 --algo 160000000 > $P/ncu_radix_downsweep_pair_pass1.txt
python profiles/ncu_summary.py $R --kernel radix_downsweep --traffic-json $P/traffic_radix_downsweep_powerlaw_1m_10m.json
python profiles/ncu_summary.py $R --kernel gather_s --algo 720000000 > $P/ncu_gather_s.txt
python profiles/ncu_summary.py $R --kernel gather_p --algo 400000000 > $P/ncu_gather_p.txt
for k in forward_scatter star_filter pack_edges radix_upsweep pair_keys star_work tri_wedge tri_filter; do
  python profiles/ncu_summary.py $R --kernel $k > $P/ncu_$k.txt || true
done
cp $G/bench.json $P/bench.json
cp $G/launches.csv $P/launches.csv
python profiles/summarize_launches.py $P/launches.csv > $P/launches.txt
cp $G/workstats.jsonl $P/workstats.jsonl
