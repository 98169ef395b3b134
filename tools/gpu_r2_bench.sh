# full default bench (headline + merge + mem variant + LoRA + cfg1 side measurements)
mkdir -p gpurun_out
timeout 1200 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_full.log 2>&1; echo bench rc $?
grep '^{' gpurun_out/bench_full.log | python -c "
import json,sys; d=json.loads(sys.stdin.read())
for k in ['value','ms_per_step','e2e','merge','mem_variant','lora_same_box','north_star_check','peak_hbm_gb','clocks']: print(k, d.get(k))"
tail -3 gpurun_out/bench_full.log
