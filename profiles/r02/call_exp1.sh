#!/bin/bash
# Experiment: very-long-window kernel (two-pass resolve/count vs the per-lane
# group cache) and the storage-domain time compares, A/B on one box.
set -x
out=gpurun_out/exp1; mkdir -p $out
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -x > $out/parity.log 2>&1; echo "pytest rc $?" >> $out/parity.log; tail -3 $out/parity.log
bash profiles/kab.sh 2 powerlaw_1m_10m 86400 "" ab/lib_prev.so ab/lib_old.so ab/lib_tp8.so ab/lib_tp8s256.so ab/lib_tp7s64.so > $out/kab_c1_86400.jsonl 2> $out/kab.err
bash profiles/kab.sh 1 powerlaw_50m_600m 86400 "" ab/lib_prev.so ab/lib_old.so ab/lib_tp8.so ab/lib_tp8s256.so ab/lib_tp7s64.so > $out/kab_c4_86400.jsonl 2>> $out/kab.err
bash profiles/kab.sh 2 powerlaw_50m_600m 3600 "" ab/lib_prev.so > $out/kab_c4_3600.jsonl 2>> $out/kab.err
bash profiles/kab.sh 1 triadic_25m_100m 86400 "" ab/lib_prev.so > $out/kab_c3_86400.jsonl 2>> $out/kab.err
for lib in ab/lib_stats.so ab/lib_gc8.so ab/lib_gc9.so; do
  echo "== lib ${lib:-tree}"
  TM_LIB=$lib KTIMES=1 timeout 600 python profiles/census_once.py powerlaw_1m_10m 86400 1
  TM_LIB=$lib KTIMES=1 timeout 600 python profiles/census_once.py powerlaw_50m_600m 86400 1
done > $out/cache.jsonl 2> $out/cache.err
ncu --set full --clock-control none --import-source on -k regex:"tri_long|tri_window" -c 2 \
    -o $out/full_tri python profiles/census_once.py powerlaw_1m_10m 86400 1 > $out/ncu_tri.log 2>&1; echo full_tri=$?
python profiles/ncu_summary.py $out/full_tri.ncu-rep --kernel tri_window > $out/ncu_tri_window.txt
python profiles/ncu_lines.py $out/full_tri.ncu-rep "tri_window" 0.3 > $out/lines_tri_window.txt
rm -f $out/full_tri.ncu-rep
TM_LIB=ab/lib_old.so ncu --set full --clock-control none --import-source on -k regex:"tri_long" -c 2 \
    -o $out/full_old python profiles/census_once.py powerlaw_1m_10m 86400 1 > $out/ncu_old.log 2>&1; echo full_old=$?
python profiles/ncu_summary.py $out/full_old.ncu-rep --kernel tri_long --index 1 > $out/ncu_tri_long_cached_old.txt
python profiles/ncu_lines.py $out/full_old.ncu-rep "ILb1" 0.3 > $out/lines_tri_long_cached_old.txt
rm -f $out/full_old.ncu-rep
