mkdir -p gpurun_out
timeout 300 python tools/q8bench.py > gpurun_out/q8bench.txt 2>&1; echo q8b $?
timeout 300 python tools/microbench.py gemm > gpurun_out/microbench_gemm_ms.txt 2>&1; echo mb $?
timeout 1800 python -m pytest tests -q -m gpu --timeout 900 -rf > gpurun_out/gputest.log 2>&1; echo tests $?
rm -f gpurun_out/q8_configs.jsonl
for c in 8b-poetx-mem 8b-poetxq-mem 1b-poetx-mem 1b-poetxq-mem; do timeout 600 python tools/configs_bench.py --one $c >> gpurun_out/q8_configs.jsonl 2>>gpurun_out/q8_configs.err; done
timeout 600 python bench.py --steps 20 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/bench_smem.log 2>&1
cat gpurun_out/q8bench.txt gpurun_out/microbench_gemm_ms.txt; tail -3 gpurun_out/gputest.log; python -c "
import json
for l in open('gpurun_out/q8_configs.jsonl'):
    d=json.loads(l); print(d['case'], round(d.get('tokens_per_s_median_step',0)), d.get('peak_hbm_gb'), d.get('error','')[:300])"
grep '^{' gpurun_out/bench_smem.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench', d['value'], d['clocks'])"
