# final round measurements (part 2): --set full of the given kernels (regex:skip), one launch each
CMD="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline"
python build_native.py || exit 1
$CMD > /dev/null 2>&1 || exit 1
for KK in $1; do
  K=${KK%%:*}; S=${KK##*:}
  ncu --set full --clock-control none --import-source on -k regex:"$K" -s $S -c 1 -o "gpurun_out/fin_full_$K" -f $CMD > "gpurun_out/fin_ncu_$K.log" 2>&1
done
du -sh gpurun_out/*
