# 512-row pair tiles: sub-tile 0 first over the last K blocks (POETX_PAIR_TAIL) -- timeline, microbench, tests, step A/B
mkdir -p gpurun_out; rm -f gpurun_out/envab.txt
( for args in "8192 2048 2048 0 2" "8192 5632 2048 0 2"; do
    POETX_LIB_PATH=abtest/lib_trace.so timeout 120 python tools/gemmtrace.py $args | grep -v "^cta\|^entry\|setup->"
  done ) > gpurun_out/tailtrace.txt 2>&1
( echo "== tail 3"; timeout 300 python tools/microbench.py gemm
  echo "== tail 2"; POETX_LIB_PATH=abtest/lib_tail2.so timeout 300 python tools/microbench.py gemm
  echo "== tail 0"; POETX_LIB_PATH=abtest/lib_tail0.so timeout 300 python tools/microbench.py gemm ) > gpurun_out/microbench_tail.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_tc.py tests/test_gpu_q8_gemm.py tests/test_gpu_parity.py tests/test_gpu_bench_config.py tests/test_gpu_trainer.py -x -q 2>&1 | tail -2 > gpurun_out/tail_tests.txt
bash tools/gpu_envab.sh "POETX_LIB_PATH=abtest/lib_tail0.so" 3
cat gpurun_out/tailtrace.txt gpurun_out/microbench_tail.txt gpurun_out/tail_tests.txt
