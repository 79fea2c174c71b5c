set -x
python build_native.py
python -m pytest tests/test_gpu_fullsize.py -x -q -s > gpurun_out/r2_fullsize.log 2>&1; echo "fullsize rc=$?" >> gpurun_out/r2_fullsize.log
python -m pytest tests -q -m gpu --deselect tests/test_gpu_fullsize.py > gpurun_out/r2_gputests.log 2>&1; echo "gputests rc=$?" >> gpurun_out/r2_gputests.log
python bench.py --steps 20 --warmup 5 > gpurun_out/r2_bench0.json 2> gpurun_out/r2_bench0.err
tail -n 3 gpurun_out/r2_fullsize.log gpurun_out/r2_gputests.log
