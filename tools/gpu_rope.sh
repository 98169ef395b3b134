mkdir -p gpurun_out
( timeout 600 python -m pytest tests/test_gpu_rowops.py tests/test_gpu_trainer.py -q -m gpu -x 2>&1 | tail -2
  for i in 1 2; do timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('bench', d['value'], d['ms_per_step'])"; done
  timeout 600 python tools/profile_step.py --serial --rows 40 2>&1 | grep -E "rope|step wall"
) > gpurun_out/rope.txt 2>&1
