# fused CNP change: parity, microbench, bench
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_cnp_fused.py tests/test_gpu_bench_config.py tests/test_gpu_trainer.py tests/test_gpu_parity.py -q -m gpu -x -rf > gpurun_out/cnp_tests.log 2>&1; echo tests $?
timeout 300 python tools/cnpbench.py > gpurun_out/cnpbench.log 2>&1; echo cnpbench $?
timeout 600 python bench.py --steps 10 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/bench_cnp.log 2>&1; echo bench $?
tail -3 gpurun_out/cnp_tests.log; cat gpurun_out/cnpbench.log; grep '^{' gpurun_out/bench_cnp.log | cut -c1-400
