set -x
mkdir -p gpurun_out/r02
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -m gpu -q -x -k "not triadic" > gpurun_out/r02/gputest7.log 2>&1; echo "pytest rc $?" >> gpurun_out/r02/gputest7.log
for d in 3600 86400; do KTIMES=1 timeout 600 python profiles/census_once.py powerlaw_50m_600m $d 2; done > gpurun_out/r02/c4_gc.jsonl 2> gpurun_out/r02/c4_gc.err
