set -x
G=gpurun_out/s10; mkdir -p $G
python profiles/census_once.py powerlaw_50m_600m 3600 1 > $G/once.log 2>&1; echo once=$?
ncu --set full --clock-control none --import-source on -k regex:"radix_downsweep" -c 8 \
    -o $G/full_sort python profiles/census_once.py powerlaw_50m_600m 3600 1 > $G/ncu_sort.log 2>&1; echo full_sort=$?
NODE_ALGO=(28800000000 38400000000 38400000000 38400000000)
PAIR_ALGO=(19200000000 19200000000 19200000000 21600000000)
for i in 0 1 2 3; do
  python profiles/ncu_summary.py $G/full_sort.ncu-rep --kernel radix_downsweep --index $i --algo ${NODE_ALGO[$i]} \
    > $G/ncu_radix_downsweep_node_pass$((i+1)).txt
  python profiles/ncu_summary.py $G/full_sort.ncu-rep --kernel radix_downsweep --index $((i+4)) --algo ${PAIR_ALGO[$i]} \
    > $G/ncu_radix_downsweep_pair_pass$((i+1)).txt
done
python profiles/ncu_lines.py $G/full_sort.ncu-rep radix_downsweep > $G/lines_radix_downsweep.txt
ncu -i $G/full_sort.ncu-rep --page source --csv --print-source sass > $G/sass_sort.csv 2>/dev/null; gzip -f $G/sass_sort.csv
ls -la $G
rm -f $G/full_sort.ncu-rep
