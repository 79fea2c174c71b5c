# one GPU iteration: parity (fast subset + dense/msd paths), bench, optional ncu of one kernel
# usage: bash tools/gpu_iter.sh TAG [KERNEL_REGEX]
TAG=$1; K=$2
python build_native.py || exit 1
python -m pytest tests -q -x -m gpu --deselect tests/test_gpu_fullsize.py > gpurun_out/${TAG}_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/${TAG}_tests.log
python -m pytest tests/test_gpu_fullsize.py -q -x -k "auto or slice or count" > gpurun_out/${TAG}_full.log 2>&1; echo "full rc=$?" >> gpurun_out/${TAG}_full.log
WSORT_DEBUG_TIMELINE=1 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${TAG}_timeline.json 2> gpurun_out/${TAG}_timeline.err
python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
if [ -n "$K" ]; then
  python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:$K -s 1 -c 1 -o gpurun_out/${TAG}_prof -f \
      python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/${TAG}_ncu.log 2>&1
fi
tail -n 2 gpurun_out/${TAG}_tests.log gpurun_out/${TAG}_full.log
