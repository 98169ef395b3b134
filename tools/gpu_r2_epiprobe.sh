# what bounds the pair-GEMM epilogue: sub-tile release times, with and without the stores
mkdir -p gpurun_out
( for v in trace trace_nostore; do
    for args in "8192 2048 2048 0 2" "8192 2048 2048 0 1" "8192 5632 2048 0 2"; do
      echo "== $v"; POETX_LIB_PATH=abtest/lib_$v.so timeout 120 python tools/gemmtrace.py $args | grep -v "^cta\|^entry\|setup->"
    done
  done ) > gpurun_out/epiprobe2.txt 2>&1
cat gpurun_out/epiprobe2.txt
