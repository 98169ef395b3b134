mkdir -p gpurun_out
for pct in 100 50 25 1; do POETX_OUTER_SM_PCT=$pct timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_pct$pct.log 2>&1; done
