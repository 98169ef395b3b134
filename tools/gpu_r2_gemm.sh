# pair GEMM 512x256 tiles: correctness + microbench + bench
mkdir -p gpurun_out
timeout 600 python tools/microbench.py gemm > gpurun_out/microbench_gemm_ms.txt 2>&1; echo mb $?
timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_parity.py tests/test_gpu_bench_config.py -q -m gpu -x -rf > gpurun_out/gemm_tests.log 2>&1; echo tests $?
timeout 600 python bench.py --steps 10 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/bench_ms2.log 2>&1; echo bench $?
POETX_PAIR_MS=1 timeout 600 python bench.py --steps 10 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/bench_ms1.log 2>&1; echo bench1 $?
cat gpurun_out/microbench_gemm_ms.txt; tail -3 gpurun_out/gemm_tests.log
for f in bench_ms2 bench_ms1; do grep '^{' gpurun_out/$f.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$f', d['value'], d['clocks']['sm_mhz'], d['roofline']['achieved'], d['roofline']['frac'])"; done
