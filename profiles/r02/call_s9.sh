set -x
G=gpurun_out/s9; mkdir -p $G
timeout 2400 python -m pytest tests -m gpu -q -x > $G/gputest.log 2>&1; echo "pytest rc $?" >> $G/gputest.log
tail -3 $G/gputest.log
bash profiles/kab.sh 2 powerlaw_50m_600m 3600 "" ab/lib_nodefer.so ab/lib_defw6.so > $G/ab3600.jsonl 2>$G/ab3600.err
bash profiles/kab.sh 1 powerlaw_50m_600m 600 "" ab/lib_nodefer.so ab/lib_defw6.so > $G/ab600.jsonl 2>$G/ab600.err
bash profiles/kab.sh 1 powerlaw_50m_600m 86400 "" ab/lib_nodefer.so ab/lib_defw6.so > $G/ab86400.jsonl 2>$G/ab86400.err
bash profiles/kab.sh 1 powerlaw_1m_10m 3600 "" ab/lib_nodefer.so ab/lib_defw6.so > $G/ab_c1.jsonl 2>$G/ab_c1.err
bash profiles/kab.sh 1 triadic_25m_100m 86400 "" ab/lib_nodefer.so ab/lib_defw6.so > $G/ab_c3.jsonl 2>$G/ab_c3.err
timeout 900 python bench.py > $G/bench.json 2> $G/bench.err; echo bench=$?
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $G/launches.csv \
    python profiles/census_once.py powerlaw_50m_600m 3600 1 > $G/ncu_launch.log 2>&1; echo launches=$?
python profiles/summarize_launches.py $G/launches.csv > $G/launches.txt
grep -i downsweep $G/launches.csv | cut -c1-400 > $G/downsweep_launches.txt
