#!/bin/bash
# The GPU-side captures behind profiles/r01/ (run under gpurun), then
# profiles/refresh_r01.sh + profiles/configs_table.py here.
set -x
mkdir -p gpurun_out/r01
python bench.py > gpurun_out/r01/bench.json 2> gpurun_out/r01/bench.err; echo bench=$?
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-reader > gpurun_out/r01/ncu_launch.log 2>&1; echo launches=$?
ncu --set full --clock-control none --import-source on -k regex:"radix_downsweep|gather_s_kernel|gather_p_kernel|tri_wedge|star_work|tri_filter|star_filter|forward_scatter|pack_edges|radix_upsweep|pair_keys" -c 20 -o gpurun_out/r01/full2 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-reader > gpurun_out/r01/ncu_full.log 2>&1; echo full=$?
python profiles/workstats.py > gpurun_out/r01/workstats.jsonl 2> gpurun_out/r01/workstats.err; echo workstats=$?
bash profiles/configs_sweep.sh
