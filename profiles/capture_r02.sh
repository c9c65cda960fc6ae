#!/bin/bash
# The GPU-side captures behind profiles/r02/ (run under gpurun; each ncu pass
# only after the same command has exited 0 without ncu).  The ncu reports are
# summarised on the box (profiles/ncu_summary.py, ncu_lines.py) and deleted,
# so only text comes back; profiles/refresh_r02.sh copies it into profiles/r02.
set -x
G=gpurun_out/r02cap
mkdir -p $G
python bench.py > $G/bench.json 2> $G/bench.err; echo bench=$?
python profiles/census_once.py powerlaw_50m_600m 3600 2 > $G/census_once.jsonl 2>&1; echo once=$?
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $G/launches.csv \
    python profiles/census_once.py powerlaw_50m_600m 3600 2 > $G/ncu_launch.log 2>&1; echo launches=$?
python profiles/summarize_launches.py $G/launches.csv > $G/launches.txt
ncu --set full --clock-control none --import-source on -k regex:"radix_downsweep" -c 8 \
    -o $G/full_sort python profiles/census_once.py powerlaw_50m_600m 3600 1 > $G/ncu_sort.log 2>&1; echo full_sort=$?
# downsweep launches of one census: 4 node passes over 2m = 1.2G elements (the
# first reads the caller's src/dst/t, 8 B per element, and writes key + payload
# 16 B; the others read and write 16 B; the last writes the S columns, 16 B),
# then 4 pair passes over m = 600M (16 B + 16 B; the last writes the P columns, 20 B)
NODE_ALGO=(28800000000 38400000000 38400000000 38400000000)
PAIR_ALGO=(19200000000 19200000000 19200000000 21600000000)
for i in 0 1 2 3; do
  python profiles/ncu_summary.py $G/full_sort.ncu-rep --kernel radix_downsweep --index $i --algo ${NODE_ALGO[$i]} \
    > $G/ncu_radix_downsweep_node_pass$((i+1)).txt
  python profiles/ncu_summary.py $G/full_sort.ncu-rep --kernel radix_downsweep --index $((i+4)) --algo ${PAIR_ALGO[$i]} \
    > $G/ncu_radix_downsweep_pair_pass$((i+1)).txt
done
python profiles/ncu_summary.py $G/full_sort.ncu-rep --kernel radix_downsweep \
    --traffic-json $G/traffic_radix_downsweep_powerlaw_50m_600m_3600.json --config powerlaw_50m_600m
python profiles/ncu_lines.py $G/full_sort.ncu-rep radix_downsweep > $G/lines_radix_downsweep.txt
rm -f $G/full_sort.ncu-rep
ncu --set full --clock-control none --import-source on -k regex:"tri_mid|tri_window|tri_wedge" -c 3 \
    -o $G/full_tri python profiles/census_once.py powerlaw_50m_600m 3600 1 > $G/ncu_tri.log 2>&1; echo full_tri=$?
python profiles/ncu_summary.py $G/full_tri.ncu-rep --kernel tri_wedge > $G/ncu_tri_wedge.txt
python profiles/ncu_summary.py $G/full_tri.ncu-rep --kernel tri_mid > $G/ncu_tri_mid.txt
python profiles/ncu_summary.py $G/full_tri.ncu-rep --kernel tri_window > $G/ncu_tri_window.txt
python profiles/ncu_lines.py $G/full_tri.ncu-rep tri_wedge > $G/lines_tri_wedge.txt
python profiles/ncu_lines.py $G/full_tri.ncu-rep tri_mid > $G/lines_tri_mid.txt
rm -f $G/full_tri.ncu-rep
ncu --set full --clock-control none --import-source on \
    -k regex:"pair_keys|s_offsets|p_flags|orient_kernel|star_work|star_locate|pack_edges|forward_scatter|tri_filter|star_filter" -c 10 \
    -o $G/full_work python profiles/census_once.py powerlaw_50m_600m 3600 1 > $G/ncu_work.log 2>&1; echo full_work=$?
python profiles/ncu_summary.py $G/full_work.ncu-rep --kernel s_offsets --algo 5000000000 > $G/ncu_s_offsets.txt
python profiles/ncu_summary.py $G/full_work.ncu-rep --kernel p_flags --algo 9800000000 > $G/ncu_p_flags.txt
python profiles/ncu_summary.py $G/full_work.ncu-rep --kernel orient_kernel --algo 9750000000 > $G/ncu_orient.txt
python profiles/ncu_summary.py $G/full_work.ncu-rep --kernel pack_edges --algo 9600000000 > $G/ncu_pack_edges.txt
python profiles/ncu_summary.py $G/full_work.ncu-rep --kernel pair_keys --algo 28800000000 > $G/ncu_pair_keys.txt
for k in forward_scatter tri_filter star_filter star_locate star_work; do
  python profiles/ncu_summary.py $G/full_work.ncu-rep --kernel $k > $G/ncu_$k.txt
done
python profiles/ncu_lines.py $G/full_work.ncu-rep star_work > $G/lines_star_work.txt
rm -f $G/full_work.ncu-rep
