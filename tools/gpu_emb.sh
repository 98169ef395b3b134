mkdir -p gpurun_out
b() { env "$@" timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$*', d['value'], d['ms_per_step'], d['clocks']['sm_mhz'])"; }
( for i in 1 2 3; do b POETX_FUSED_EMBED=0; b POETX_FUSED_EMBED=1; done ) > gpurun_out/emb.txt 2>&1
