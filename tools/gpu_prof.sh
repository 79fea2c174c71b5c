# ncu --set full of the given kernels, one capture each, after a plain run of the same command
# usage: bash tools/gpu_prof.sh TAG "regex1[:skip] regex2[:skip] ..." [bench args]
TAG=$1; KS=$2; shift 2
python build_native.py || exit 1
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline $*"
$CMD > gpurun_out/${TAG}_plain.json 2> gpurun_out/${TAG}_plain.err || exit 1
for KK in $KS; do
  K=${KK%%:*}; S=1; [ "$K" != "$KK" ] && S=${KK##*:}
  ncu --set full --clock-control none --import-source on -k regex:"$K" -s $S -c 1 -o gpurun_out/${TAG}_$K -f $CMD > gpurun_out/${TAG}_ncu_$K.log 2>&1
done
