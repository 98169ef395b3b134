mkdir -p gpurun_out
( POETX_LIB_PATH=abtest/lib_ctrace.so timeout 300 python tools/cnptrace.py 3696 256
  timeout 300 python tools/cnpbench.py; timeout 300 python tools/cnpbench.py 3696 128 ) > gpurun_out/cnptrace10.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_cnp_fused.py tests/test_gpu_bench_config.py -x -q 2>&1 | tail -2 >> gpurun_out/cnptrace10.txt
cat gpurun_out/cnptrace10.txt
