python build_native.py || exit 1
python -m pytest tests -q -m gpu -x > gpurun_out/r2b_t16.log 2>&1; echo "gputests rc=$?" >> gpurun_out/r2b_t16.log
python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-inflight > gpurun_out/r2b_bench_h.json 2> gpurun_out/r2b_bench_h.err
for c in 1 2; do python bench.py --config $c --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/r2b_bench_h_c$c.json 2> /dev/null; done
python tools/timeline.py 1 > gpurun_out/r2b_timeline_c1b.txt 2>&1
python tools/time_gaps.py 1 > gpurun_out/r2b_gaps_c1b.txt 2>&1
tail -n 2 gpurun_out/r2b_t16.log
