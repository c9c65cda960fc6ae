set -x
mkdir -p gpurun_out/r02
timeout 1500 python -m pytest tests/test_gpu_configs.py -m gpu -q -x -k "triadic" > gpurun_out/r02/gputest_triadic.log 2>&1; echo "pytest rc $?" >> gpurun_out/r02/gputest_triadic.log
for lib in "" profiles/ablib/lib_r9.so; do TM_LIB=$lib KTIMES=1 timeout 600 python profiles/census_once.py powerlaw_50m_600m 3600 2 | grep kernel_ms; done > gpurun_out/r02/ab_r9.jsonl 2>&1
bash profiles/capture_r02.sh
du -sh gpurun_out
