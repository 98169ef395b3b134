mkdir -p gpurun_out
( timeout 600 python -m pytest tests/test_gpu_rowops.py tests/test_gpu_trainer.py -q -m gpu -x 2>&1 | tail -2
  POETX_ROW_T8_BWD=1 timeout 600 python -m pytest tests/test_gpu_rowops.py -q -m gpu -x -k rmsnorm 2>&1 | tail -2
) > gpurun_out/t8.txt 2>&1
bash tools/gpu_ab.sh abtest/lib_prev.so 4
