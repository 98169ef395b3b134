mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_q8_gemm.py tests/test_gpu_quant.py -q -m gpu -rf > gpurun_out/q8_tests.log 2>&1; echo tests $?
rm -f gpurun_out/q8_configs.jsonl
for c in 1b-poetx-mem 1b-poetxq-mem 1b-poetx-mem 1b-poetxq-mem; do timeout 600 python tools/configs_bench.py --one $c >> gpurun_out/q8_configs.jsonl 2>>gpurun_out/q8_configs.err; done
tail -3 gpurun_out/q8_tests.log; python -c "
import json
for l in open('gpurun_out/q8_configs.jsonl'):
    d=json.loads(l); print(d['case'], round(d.get('tokens_per_s_median_step',0)), d.get('peak_hbm_gb'), d.get('error','')[:300])"
