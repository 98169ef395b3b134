mkdir -p gpurun_out
( for lib in "" abtest/lib_bd51.so abtest/lib_bd41.so; do
    for a in "2048 0" "2048 1" "5632 0" "5632 1"; do echo "${lib:-current} $(POETX_LIB_PATH=$lib timeout 120 python tools/blockbench.py apply $a --time 2>&1 | tail -1)"; done
  done
) > gpurun_out/bd.txt 2>&1
