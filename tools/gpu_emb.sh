mkdir -p gpurun_out
( timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
  timeout 300 python tools/profile_step.py --serial --rows 80 2>&1 | grep -E "step wall|other torch|CUDAFunctor_add"
) > gpurun_out/emb.txt 2>&1
