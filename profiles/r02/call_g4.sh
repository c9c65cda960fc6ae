# The reference's run_parallel on the whole config 4 on the box's host cores
# (background), ncu captures of the delta-86400 top kernels on the GPU meanwhile.
set -x
out=gpurun_out/g4; mkdir -p $out
free -g > $out/free.txt; nproc >> $out/free.txt
(GOLDEN_OUT=$out GOLDEN_DELTAS=${1:-600,3600} timeout ${2:-3900} python tests/golden/make_golden.py --only-extra --config4-full \
   > $out/golden.log 2>&1; echo "golden rc $?" >> $out/golden.log) &
GP=$!
sleep 240   # generation on the GPU first
KTIMES=1 timeout 900 python profiles/census_once.py powerlaw_50m_600m 86400 1 > $out/once86400.jsonl 2>&1; echo once=$?
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"tri_mid|tri_window|tri_wedge" -c 3 \
    -o $out/full_tri86400 python profiles/census_once.py powerlaw_50m_600m 86400 1 > $out/ncu_tri86400.log 2>&1; echo ncu=$?
for k in tri_mid tri_window tri_wedge; do
  python profiles/ncu_summary.py $out/full_tri86400.ncu-rep --kernel $k > $out/ncu_${k}_86400.txt
  python profiles/ncu_lines.py $out/full_tri86400.ncu-rep $k > $out/lines_${k}_86400.txt
done
rm -f $out/full_tri86400.ncu-rep
free -g >> $out/free.txt
wait $GP
tail -5 $out/golden.log
