mkdir -p gpurun_out
( for db in 0 1 0 1; do POETX_ROW_DB=$db timeout 120 python tools/rowbench.py swiglu_bwd --time; done
  timeout 300 python -m pytest tests/test_gpu_rowops.py -q -m gpu 2>&1 | tail -2
  for db in 0 1; do POETX_ROW_DB=$db timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('ROW_DB=$db', d['value'], d['ms_per_step'])"; done
) > gpurun_out/ab_row.txt 2>&1
