# K1 experiments: variants built by tools/build_variant.py (WSORT_IG_PIECE / _MODE: work distribution inside a CTA;
# WSORT_IG_THREADS / WSORT_IG_MINB: warps per CTA, CTAs per SM; WSORT_IG_CACHE_LG: hash-cache slots; WSORT_IG_EVICT),
# k1_ingest mean launch time on config 4
(
for V in ev0 t896 t768; do WSORT_LIB=build/var_$V/libwsort.so python tools/time_k1.py 0; done
python tools/time_k1.py 0
) > gpurun_out/p_k1g.txt 2>&1
