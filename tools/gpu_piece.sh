# K1 experiments: k1_ingest mean launch time on config 4 for variants built by tools/build_variant.py, then the in-tree
# build. usage (on the GPU box): bash tools/gpu_piece.sh TAG VARIANT...   -> gpurun_out/k1_TAG.txt
# Switches (k_ingest.cu / wsort_internal.cuh): WSORT_IG_PIECE / WSORT_IG_PIECE_MODE (work distribution inside a CTA),
# WSORT_IG_THREADS / WSORT_IG_MINB (warps per CTA, CTAs per SM), WSORT_IG_CACHE_LG (hash-cache slots), WSORT_IG_EVICT.
# e.g. python tools/build_variant.py m1c12 "k_ingest.cu:-DWSORT_IG_MINB=1 -DWSORT_IG_THREADS=1024 -DWSORT_IG_CACHE_LG=12"
TAG=$1; shift
(
for V in "$@"; do WSORT_LIB=build/var_$V/libwsort.so python tools/time_k1.py 0; done
python tools/time_k1.py 0
) > gpurun_out/k1_$TAG.txt 2>&1
