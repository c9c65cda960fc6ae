set -x
G=gpurun_out/s6; mkdir -p $G
bash profiles/kab.sh 2 powerlaw_50m_600m 3600 "" ab/lib_w6.so ab/lib_w8.so ab/lib_l8.so ab/lib_mw32.so ab/lib_mw16.so > $G/ab3600.jsonl 2>$G/ab3600.err
bash profiles/kab.sh 1 powerlaw_50m_600m 86400 "" ab/lib_mw32.so ab/lib_mw16.so ab/lib_c5.so ab/lib_c6.so > $G/ab86400.jsonl 2>$G/ab86400.err
ncu --set full --clock-control none --import-source on -k regex:"tri_window" -c 1 \
    -o $G/full_win1 python profiles/census_once.py powerlaw_1m_10m 86400 1 > $G/ncu_win1.log 2>&1; echo $?
python profiles/ncu_summary.py $G/full_win1.ncu-rep --kernel tri_window > $G/ncu_tri_window_c1.txt
python profiles/ncu_lines.py $G/full_win1.ncu-rep tri_window > $G/lines_tri_window_c1.txt
rm -f $G/full_win1.ncu-rep
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"tri_window" -c 1 \
    -o $G/full_win4 python profiles/census_once.py powerlaw_50m_600m 86400 1 > $G/ncu_win4.log 2>&1; echo $?
python profiles/ncu_summary.py $G/full_win4.ncu-rep --kernel tri_window > $G/ncu_tri_window_c4.txt
python profiles/ncu_lines.py $G/full_win4.ncu-rep tri_window > $G/lines_tri_window_c4.txt
rm -f $G/full_win4.ncu-rep
