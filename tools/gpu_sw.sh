mkdir -p gpurun_out
( timeout 600 python -m pytest tests/test_gpu_rowops.py tests/test_gpu_trainer.py -q -m gpu -x 2>&1 | tail -2
  for lib in abtest/lib_prev.so ""; do POETX_LIB_PATH=$lib timeout 120 python tools/rowbench.py swiglu_bwd --time 2>&1 | tail -1; done
) > gpurun_out/sw.txt 2>&1
bash tools/gpu_ab.sh abtest/lib_prev.so 3
