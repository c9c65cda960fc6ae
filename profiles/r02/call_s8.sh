set -x
G=gpurun_out/s8; mkdir -p $G
nproc > $G/host.txt; free -g >> $G/host.txt
timeout 2400 python -m pytest tests -m gpu -q -x > $G/gputest.log 2>&1; echo "pytest rc $?" >> $G/gputest.log
tail -3 $G/gputest.log
timeout 900 python bench.py > $G/bench.json 2> $G/bench.err; echo bench=$?
TM_H2D_PACK=0 timeout 900 python bench.py --no-cpu-baseline > $G/bench_nopack.json 2> $G/bench_nopack.err; echo bench=$?
for d in 3600 600 86400; do KTIMES=1 timeout 600 python profiles/census_once.py powerlaw_50m_600m $d 2; done > $G/c4.jsonl 2> $G/c4.err
TM_RAW_FIRST=0 KTIMES=1 timeout 600 python profiles/census_once.py powerlaw_50m_600m 3600 2 > $G/c4_noraw.jsonl 2>&1
KTIMES=1 timeout 600 python profiles/census_once.py triadic_25m_100m 86400 2 > $G/c3.jsonl 2>&1
KTIMES=1 timeout 600 python profiles/census_once.py powerlaw_1m_10m 3600 2 > $G/c1.jsonl 2>&1
