# the paper's data-structure comparison (Table 1): ragged references ("vectors of strings") vs
# fixed-width keys ("array char 3D"), same sort family (odd-even transposition / bitonic tiles + merge path)
for c in 1 2 3; do
  for a in ragged oets_merge auto; do
    python bench.py --config $c --algo $a --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${1}_c${c}_$a.json 2> gpurun_out/${1}_c${c}_$a.err
  done
done
