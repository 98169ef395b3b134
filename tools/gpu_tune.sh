# same-box A/B of env toggles: bash tools/gpu_tune.sh "POETX_X=1" "POETX_ATTN_BWD=0" ...  (2 rounds)
mkdir -p gpurun_out
b() { env "$@" timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$*', d['value'], d['ms_per_step'], d['clocks']['sm_mhz'])"; }
( for i in 1 2 3; do for e in "$@"; do b $e; done; done ) > gpurun_out/tune.txt 2>&1
