mkdir -p gpurun_out
timeout 300 python tools/q8bench.py 2>&1 | tail -12
rm -f gpurun_out/q8_configs.jsonl
for c in 8b-poetxq-mem 8b-poetx-mem; do timeout 600 python tools/configs_bench.py --one $c >> gpurun_out/q8_configs.jsonl 2>>gpurun_out/q8_configs.err; done
POETX_Q8_GEMM=2 timeout 600 python tools/configs_bench.py --one 8b-poetxq-mem >> gpurun_out/q8_configs.jsonl 2>>gpurun_out/q8_configs.err
python -c "
import json
for l in open('gpurun_out/q8_configs.jsonl'):
    d=json.loads(l); print(d['case'], round(d.get('tokens_per_s_median_step',0)), d.get('peak_hbm_gb'), d.get('error','')[:300])"
