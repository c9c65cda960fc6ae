set -x
mkdir -p gpurun_out/s5
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/s5/gputest.log 2>&1; echo "pytest rc $?" >> gpurun_out/s5/gputest.log
timeout 600 python bench.py > gpurun_out/s5/bench.json 2> gpurun_out/s5/bench.err; echo bench=$?
for d in 600 3600 86400; do KTIMES=1 timeout 600 python profiles/census_once.py powerlaw_50m_600m $d 2; done > gpurun_out/s5/c4.jsonl 2> gpurun_out/s5/c4.err
KTIMES=1 timeout 600 python profiles/census_once.py triadic_25m_100m 86400 2 > gpurun_out/s5/c3.jsonl 2>&1
KTIMES=1 timeout 600 python profiles/census_once.py powerlaw_1m_10m 86400 2 > gpurun_out/s5/c1.jsonl 2>&1
