mkdir -p gpurun_out
( POETX_LIB_PATH=abtest/lib_ctrace.so timeout 300 python tools/cnptrace.py 3696 256
  timeout 300 python tools/cnpbench.py; timeout 300 python tools/cnpbench.py 3696 128 ) > gpurun_out/cnptrace8.txt 2>&1
cat gpurun_out/cnptrace8.txt
