# final round measurements (part 1): bench (N=1 default), reference arm, ncu launch list and per-kernel DRAM
# traffic of one step. Part 2 (tools/gpu_final_full.sh): --set full captures of the top kernels.
set -x
python build_native.py || exit 1
python bench.py --steps 20 --warmup 5 > gpurun_out/fin_bench.json 2> gpurun_out/fin_bench.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/fin_ref.json 2> gpurun_out/fin_ref.err
CMD="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline"
$CMD > /dev/null 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fin_launches.csv $CMD > gpurun_out/fin_ncu1.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/fin_traffic.csv $CMD > gpurun_out/fin_ncu2.log 2>&1
du -sh gpurun_out/*
