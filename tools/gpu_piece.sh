# K1 work-distribution experiments (WSORT_IG_PIECE / WSORT_IG_PIECE_MODE variants built by tools/build_variant.py)
(
WSORT_LIB=build/var_rr8/libwsort.so python tools/time_k1.py 0
WSORT_LIB=build/var_rr64/libwsort.so python tools/time_k1.py 0
WSORT_LIB=build/var_contig/libwsort.so python tools/time_k1.py 256 512 1024 4096
python tools/time_k1.py 0
) > gpurun_out/p_k1b.txt 2>&1
