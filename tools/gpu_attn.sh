mkdir -p gpurun_out
( for lib in abtest/lib_prev.so "" abtest/lib_prev.so ""; do echo "${lib:-current}: $(POETX_LIB_PATH=$lib timeout 120 python tools/attnbench.py 2>&1 | tail -1)"; done
) > gpurun_out/attn_prof.txt 2>&1
