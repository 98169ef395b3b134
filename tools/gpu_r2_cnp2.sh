# fused CNP scatter rework -- phase trace, standalone timing, tests
mkdir -p gpurun_out
POETX_LIB_PATH=abtest/lib_ctrace.so timeout 300 python tools/cnptrace.py 3696 256 > gpurun_out/cnptrace6.txt 2>&1
POETX_LIB_PATH=abtest/lib_ctrace.so timeout 300 python tools/cnptrace.py 3696 128 >> gpurun_out/cnptrace6.txt 2>&1
( for v in "" cnp_old; do
    echo "== ${v:-new}"; POETX_LIB_PATH=${v:+abtest/lib_$v.so} timeout 300 python tools/cnpbench.py; POETX_LIB_PATH=${v:+abtest/lib_$v.so} timeout 300 python tools/cnpbench.py 3696 128
  done ) > gpurun_out/cnpbench6.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_cnp_fused.py tests/test_gpu_tc.py tests/test_gpu_bench_config.py tests/test_gpu_parity.py -x -q 2>&1 | tail -3 > gpurun_out/cnp6_tests.txt
cat gpurun_out/cnptrace6.txt gpurun_out/cnpbench6.txt gpurun_out/cnp6_tests.txt
