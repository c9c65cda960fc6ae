# The reference's run_parallel on the whole config 4 on the box's host cores
# (background; ~130 GB of host memory at its peak), the small-graph GPU parity
# tests and occupancy A/B runs of the triangle kernels on the GPU meanwhile.
set -x
out=gpurun_out/g4; mkdir -p $out
free -g > $out/free.txt; nproc >> $out/free.txt
(GOLDEN_OUT=$out GOLDEN_DELTAS=${1:-600,3600} timeout ${2:-3900} python tests/golden/make_golden.py --only-extra --config4-full \
   > $out/golden.log 2>&1; echo "golden rc $?" >> $out/golden.log) &
GP=$!
sleep 200   # generation on the GPU first
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x > $out/parity.log 2>&1; echo "pytest rc $?" >> $out/parity.log
bash profiles/kab.sh 2 powerlaw_50m_600m 3600 "" ab/lib_w6.so ab/lib_w8.so ab/lib_l8.so ab/lib_w6l8.so > $out/kab3600.jsonl 2> $out/kab.err
bash profiles/kab.sh 1 powerlaw_50m_600m 86400 "" ab/lib_l8.so ab/lib_w6l8.so > $out/kab86400.jsonl 2>> $out/kab.err
bash profiles/kab.sh 1 powerlaw_50m_600m 600 "" ab/lib_w6l8.so > $out/kab600.jsonl 2>> $out/kab.err
free -g >> $out/free.txt
wait $GP
free -g >> $out/free.txt
tail -5 $out/golden.log
