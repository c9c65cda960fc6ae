set -x
G=gpurun_out/s7; mkdir -p $G gpurun_out/g4
nproc > $G/host.txt; free -g >> $G/host.txt
# the reference's run_parallel on the whole config 4 on the host cores, in the background
(GOLDEN_OUT=gpurun_out/g4 GOLDEN_DELTAS=${GOLDEN_DELTAS:-600} timeout 5000 python tests/golden/make_golden.py --only-extra --config4-full \
   > gpurun_out/g4/golden.log 2>&1; echo "golden rc $?" >> gpurun_out/g4/golden.log) &
GP=$!
sleep 90
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x > $G/gputest.log 2>&1; echo "pytest rc $?" >> $G/gputest.log
bash profiles/kab.sh 2 powerlaw_50m_600m 3600 "" ab/lib_nomid.so ab/lib_mid8.so ab/lib_nomid8.so > $G/ab3600.jsonl 2>$G/ab3600.err
bash profiles/kab.sh 1 powerlaw_50m_600m 600 "" ab/lib_nomid.so ab/lib_mid8.so ab/lib_nomid8.so > $G/ab600.jsonl 2>$G/ab600.err
bash profiles/kab.sh 1 powerlaw_50m_600m 86400 "" ab/lib_nomid.so ab/lib_mid8.so ab/lib_nomid8.so > $G/ab86400.jsonl 2>$G/ab86400.err
bash profiles/kab.sh 1 powerlaw_1m_10m 3600 "" ab/lib_nomid.so ab/lib_mid8.so ab/lib_nomid8.so > $G/ab_c1.jsonl 2>$G/ab_c1.err
bash profiles/kab.sh 1 triadic_25m_100m 86400 "" ab/lib_nomid.so ab/lib_mid8.so ab/lib_nomid8.so > $G/ab_c3.jsonl 2>$G/ab_c3.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"tri_mid" -c 1 \
    -o $G/full_mid python profiles/census_once.py powerlaw_50m_600m 3600 1 > $G/ncu_mid.log 2>&1; echo $?
python profiles/ncu_summary.py $G/full_mid.ncu-rep --kernel tri_mid > $G/ncu_tri_mid_c4.txt
python profiles/ncu_lines.py $G/full_mid.ncu-rep tri_mid > $G/lines_tri_mid_c4.txt
rm -f $G/full_mid.ncu-rep
free -g >> $G/host.txt
wait $GP
tail -5 gpurun_out/g4/golden.log
