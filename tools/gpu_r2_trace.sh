# pair-GEMM timelines (build-time probe) at the Llama-1B shapes
mkdir -p gpurun_out
export POETX_LIB_PATH=abtest/lib_trace.so
( for args in "8192 2048 2048 0 2" "8192 2048 2048 0 1" "8192 2048 2048 1 2" "8192 5632 2048 0 2" "8192 2048 5632 0 2"; do
    timeout 120 python tools/gemmtrace.py $args
    echo
  done ) > gpurun_out/gemmtrace.txt 2>&1
cat gpurun_out/gemmtrace.txt
