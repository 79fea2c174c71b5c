python build_native.py || exit 1
python tools/time_k1.py 0 > gpurun_out/r2b_k1_c2.txt 2>&1
WSORT_LIB=build/var_c2/libwsort.so python tools/time_k1.py 0 >> gpurun_out/r2b_k1_c2.txt 2>&1
python tools/time_k1.py 0 >> gpurun_out/r2b_k1_c2.txt 2>&1
WSORT_LIB=build/var_c2/libwsort.so python tools/time_k1.py 0 >> gpurun_out/r2b_k1_c2.txt 2>&1
