mkdir -p gpurun_out
POETX_PAIR_DIRECT_EPI=1 timeout 300 python -m pytest tests/test_gpu_tc.py -x -q > gpurun_out/epi_tests.log 2>&1; echo "rc=$?" >> gpurun_out/epi_tests.log
for e in 0 1; do POETX_PAIR_DIRECT_EPI=$e timeout 300 python tools/microbench.py gemm > gpurun_out/mb_gemm_epi$e.txt 2>&1; done
for e in 0 1; do POETX_PAIR_DIRECT_EPI=$e timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_epi$e.log 2>&1; done
