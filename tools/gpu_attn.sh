mkdir -p gpurun_out
( timeout 300 python -m pytest tests/test_gpu_attention.py -q -m gpu -x 2>&1 | tail -3
  timeout 120 python tools/attnbench.py
  for m in 0 1 0 1; do POETX_ATTN_BWD=$m timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('ATTN_BWD=$m', d['value'], d['ms_per_step'])"; done
) > gpurun_out/attn_prof.txt 2>&1
