mkdir -p gpurun_out
POETX_LIB_PATH=abtest/lib_ctrace.so timeout 300 python tools/cnptrace.py 3696 256 > gpurun_out/cnptrace5.txt 2>&1
cat gpurun_out/cnptrace5.txt
