mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke $?
timeout 1800 python -m pytest tests -q -m gpu --timeout 900 -rf > gpurun_out/gputest.log 2>&1; echo tests $?
timeout 1200 python bench.py --steps 20 --warmup 3 > gpurun_out/bench_full.log 2>&1; echo bench $?
rm -f gpurun_out/q8_configs.jsonl
for c in 1b-poetxq-mem 8b-poetxq-mem 8b-poetx-mem 1b-lora; do timeout 600 python tools/configs_bench.py --one $c >> gpurun_out/q8_configs.jsonl 2>>gpurun_out/q8_configs.err; done
tail -2 gpurun_out/smoke.log; tail -3 gpurun_out/gputest.log
grep '^{' gpurun_out/bench_full.log | python -c "
import json,sys; d=json.loads(sys.stdin.read())
for k in ['value','ms_per_step','e2e','roofline','step_tc_roofline','merge','mem_variant','xq_variant','lora_same_box','north_star_check','peak_hbm_gb','clocks']: print(k, d.get(k))"
python -c "
import json
for l in open('gpurun_out/q8_configs.jsonl'):
    d=json.loads(l); print(d['case'], round(d.get('tokens_per_s_median_step',0)), d.get('peak_hbm_gb'), d.get('error','')[:300])"
