# bench lines for BASELINE configs 1-3 (parity-size inputs; 1-2 are latency-bound) next to config 4
for c in 1 2 3; do
  python bench.py --config $c --steps 20 --warmup 5 --no-e2e > gpurun_out/${1}_c$c.json 2> gpurun_out/${1}_c$c.err
done
