for L in ab/lib_prev.so ab/lib_l6.so ab/lib_l4.so; do echo $L; TM_LIB=$L python profiles/config4_tri.py; done
