mkdir -p gpurun_out
( timeout 600 python -m pytest tests/test_gpu_tc.py tests/test_gpu_parity.py -q -m gpu -x 2>&1 | tail -2
  for lib in abtest/lib_prev.so "" ; do
    for a in "2048 0" "2048 1" "5632 0" "5632 1"; do echo "${lib:-current} $(POETX_LIB_PATH=$lib timeout 120 python tools/blockbench.py apply $a --time 2>&1 | tail -1)"; done
  done
) > gpurun_out/bd.txt 2>&1
bash tools/gpu_ab.sh abtest/lib_prev.so 3
