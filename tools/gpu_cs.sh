mkdir -p gpurun_out
( timeout 600 python -m pytest tests/test_gpu_rowops.py tests/test_gpu_trainer.py -q -m gpu -x 2>&1 | tail -2
  timeout 600 python tools/profile_step.py --serial --rows 70 2>&1 | grep -E "step wall|colsum"
) > gpurun_out/cs.txt 2>&1
bash tools/gpu_ab.sh abtest/lib_prev.so 3
