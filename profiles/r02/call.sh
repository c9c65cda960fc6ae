set -x
mkdir -p gpurun_out/r02
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r02/gputest15.log 2>&1; echo "pytest rc $?" >> gpurun_out/r02/gputest15.log
for d in 3600 86400; do KTIMES=1 timeout 600 python profiles/census_once.py powerlaw_50m_600m $d 2; done > gpurun_out/r02/c4_occ6.jsonl 2> gpurun_out/r02/c4_occ6.err
