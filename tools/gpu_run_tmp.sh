python build_native.py || exit 1
python tools/time_k1.py 0 > gpurun_out/r2b_k1_late.txt 2>&1
WSORT_LIB=build/var_late/libwsort.so python tools/time_k1.py 0 1 >> gpurun_out/r2b_k1_late.txt 2>&1
python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2b_bench_inflight.json 2> gpurun_out/r2b_bench_inflight.err
