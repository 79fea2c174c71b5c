python build_native.py || exit 1
for i in 1 2; do
python -m pytest tests/test_gpu_fullsize.py -x -q > gpurun_out/r2b_full4_$i.log 2>&1; echo "fullsize rc=$?" >> gpurun_out/r2b_full4_$i.log
done
python -m pytest tests -q -m gpu -x --deselect tests/test_gpu_fullsize.py > gpurun_out/r2b_t12.log 2>&1; echo "gputests rc=$?" >> gpurun_out/r2b_t12.log
python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2b_bench_g.json 2> gpurun_out/r2b_bench_g.err; echo "rc=$?" >> gpurun_out/r2b_bench_g.err
tail -n 2 gpurun_out/r2b_full4_*.log gpurun_out/r2b_t12.log gpurun_out/r2b_bench_g.err
