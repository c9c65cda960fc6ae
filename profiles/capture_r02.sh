#!/bin/bash
# The GPU-side captures behind profiles/r02/ (run under gpurun; each ncu pass
# only after the same command has exited 0 without ncu).
set -x
mkdir -p gpurun_out/r02cap
python bench.py > gpurun_out/r02cap/bench.json 2> gpurun_out/r02cap/bench.err; echo bench=$?
python profiles/census_once.py powerlaw_50m_600m 3600 2 > gpurun_out/r02cap/census_once.jsonl 2>&1; echo once=$?
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02cap/launches.csv \
    python profiles/census_once.py powerlaw_50m_600m 3600 2 > gpurun_out/r02cap/ncu_launch.log 2>&1; echo launches=$?
ncu --set full --clock-control none --import-source on -k regex:"radix_downsweep" -c 2 \
    -o gpurun_out/r02cap/full_sort python profiles/census_once.py powerlaw_50m_600m 3600 1 > gpurun_out/r02cap/ncu_sort.log 2>&1; echo full_sort=$?
ncu --set full --clock-control none --import-source on \
    -k regex:"tri_long|tri_wedge|pair_keys|gather_s_pay|gather_p_pay|star_work|star_locate|pack_edges|radix_upsweep|forward_scatter|tri_filter" -c 12 \
    -o gpurun_out/r02cap/full_work python profiles/census_once.py powerlaw_50m_600m 3600 1 > gpurun_out/r02cap/ncu_work.log 2>&1; echo full_work=$?
