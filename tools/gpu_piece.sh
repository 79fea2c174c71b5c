# K1 experiments: variants built by tools/build_variant.py (WSORT_IG_PIECE / _MODE: work distribution inside a CTA;
# WSORT_IG_THREADS / WSORT_IG_MINB: warps per CTA, CTAs per SM; WSORT_IG_CACHE_LG: hash-cache slots), k1_ingest mean
# launch time on config 4; then the GPU tests and the bench of the in-tree build
python tools/time_k1.py 0 > gpurun_out/p_k1f.txt 2>&1
python -m pytest tests -q -m gpu > gpurun_out/p_tests3.log 2>&1; echo "rc=$?" >> gpurun_out/p_tests3.log
python __graft_entry__.py smoke > gpurun_out/p_smoke3.log 2>&1
for i in 0 1; do python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-inflight > gpurun_out/p_bench3_$i.json 2>&1; done
for c in 1 2 3; do python bench.py --config $c --steps 20 --warmup 5 --no-e2e > gpurun_out/p_c$c.json 2>&1; done
WSORT_STRESS_REPS=3 python tools/stress_run.py edge > gpurun_out/p_stress_edge.txt 2>&1
WSORT_STRESS_REPS=3 python tools/stress_run.py mid auto auto_count lsd_radix > gpurun_out/p_stress_mid.txt 2>&1
