python build_native.py || exit 1
python -m pytest tests/test_gpu_fullsize.py -x -q > gpurun_out/r2b_full1.log 2>&1; echo "fullsize rc=$?" >> gpurun_out/r2b_full1.log
python -m pytest tests -q -m gpu -x --deselect tests/test_gpu_fullsize.py > gpurun_out/r2b_t10.log 2>&1; echo "gputests rc=$?" >> gpurun_out/r2b_t10.log
tail -2 gpurun_out/r2b_full1.log gpurun_out/r2b_t10.log
