# round-2 final measurements (r02e: final K1): bench + reference arm + configs 1-3, launch list, per-kernel
# DRAM traffic of one step, --set full of the top kernels, GPU test logs
set -x
python build_native.py || exit 1
python -m pytest tests -q -m gpu > gpurun_out/f5_gputests.log 2>&1; echo "gputests rc=$?" >> gpurun_out/f5_gputests.log
python bench.py --steps 20 --warmup 5 > gpurun_out/f5_bench.json 2> gpurun_out/f5_bench.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/f5_ref.json 2> gpurun_out/f5_ref.err
for c in 1 2 3; do python bench.py --config $c --steps 20 --warmup 5 --no-e2e > gpurun_out/f5_c$c.json 2> gpurun_out/f5_c$c.err; done
CMD="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-inflight"
$CMD > /dev/null 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/f5_launches.csv $CMD > gpurun_out/f5_ncu1.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/f5_traffic.csv $CMD > gpurun_out/f5_ncu2.log 2>&1
for KK in k_ingest:1 k_msd_scatter0:1 "k_msd_fin$:0"; do
  K=${KK%%:*}; S=${KK##*:}
  ncu --set full --clock-control none --import-source on -k regex:"$K" -s $S -c 1 -o "gpurun_out/f5_full_$K" -f $CMD > "gpurun_out/f5_ncu_$K.log" 2>&1
done
du -sh gpurun_out/f5_*
