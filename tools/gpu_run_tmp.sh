python build_native.py || exit 1
python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2b_bench_hp.json 2> gpurun_out/r2b_bench_hp.err
WSORT_NO_HP=1 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2b_bench_nohp.json 2> gpurun_out/r2b_bench_nohp.err
python tools/timeline.py 4 > gpurun_out/r2b_timeline_hp.txt 2>&1
python -m pytest tests -q -m gpu -x --deselect tests/test_gpu_fullsize.py > gpurun_out/r2b_t13.log 2>&1; echo "gputests rc=$?" >> gpurun_out/r2b_t13.log
tail -n 2 gpurun_out/r2b_t13.log
