# K1 experiments: variants built by tools/build_variant.py (WSORT_IG_PIECE / _MODE: work distribution inside a CTA;
# WSORT_IG_THREADS: warps per CTA), k1_ingest mean launch time on config 4
(
for T in 320 384 448 576 640; do WSORT_LIB=build/var_thr$T/libwsort.so python tools/time_k1.py 0; done
python tools/time_k1.py 0
) > gpurun_out/p_k1c.txt 2>&1
