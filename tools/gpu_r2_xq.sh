mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_q8_gemm.py -q -m gpu -rf 2>&1 | tail -2
timeout 300 python tools/q8bench.py 2>&1 | tail -4
for i in 1 2; do timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_xq$i.log 2>&1; grep '^{' gpurun_out/bench_xq$i.log | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print(d['value'], d['clocks']['sm_mhz']); print('mem', d.get('mem_variant')); print('xq', d.get('xq_variant'))"; done
