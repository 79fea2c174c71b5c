python build_native.py || exit 1
python -m pytest tests -q -m gpu -x > gpurun_out/r2b_t15.log 2>&1; echo "gputests rc=$?" >> gpurun_out/r2b_t15.log
for i in 1 2; do
python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-inflight > gpurun_out/r2b_bench_sub$i.json 2> /dev/null
WSORT_NO_SUBPART=1 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-inflight > gpurun_out/r2b_bench_nosub$i.json 2> /dev/null
done
python tools/timeline.py 4 > gpurun_out/r2b_timeline_sub.txt 2>&1
tail -n 2 gpurun_out/r2b_t15.log
