set -x
mkdir -p gpurun_out/r02
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/r02/gputest_final.log 2>&1; echo "pytest rc $?" >> gpurun_out/r02/gputest_final.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02/smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/r02/smoke.log
bash profiles/capture_r02.sh > gpurun_out/r02/capture.log 2>&1
bash profiles/configs_sweep.sh > gpurun_out/r02/sweep.log 2>&1
