mkdir -p gpurun_out
timeout 300 python tools/q8bench.py > gpurun_out/q8bench.txt 2>&1; echo q8b $?
timeout 900 python -m pytest tests/test_gpu_q8_gemm.py -q -m gpu -rf > gpurun_out/q8_tests.log 2>&1; echo tests $?
rm -f gpurun_out/q8_configs.jsonl
for c in 8b-poetx-mem 8b-poetxq-mem 1b-poetxq-mem; do timeout 600 python tools/configs_bench.py --one $c >> gpurun_out/q8_configs.jsonl 2>>gpurun_out/q8_configs.err; done
cat gpurun_out/q8bench.txt; tail -3 gpurun_out/q8_tests.log; python -c "
import json
for l in open('gpurun_out/q8_configs.jsonl'):
    d=json.loads(l); print(d['case'], round(d.get('tokens_per_s_median_step',0)), d.get('peak_hbm_gb'), d.get('error','')[:300])"
