python build_native.py || exit 1
python tools/timeline.py 1 > gpurun_out/r2b_timeline_c1.txt 2>&1
python tools/timeline.py 2 > gpurun_out/r2b_timeline_c2.txt 2>&1
python tools/time_gaps.py 1 > gpurun_out/r2b_gaps_c1.txt 2>&1
CMD="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline"
ncu --set full --clock-control none --import-source on -k regex:"k_msd_fin$" -s 1 -c 1 -o "gpurun_out/f2_full_k_msd_fin" -f $CMD > "gpurun_out/f2_ncu_k_msd_fin.log" 2>&1
