mkdir -p gpurun_out
b() { env "$@" timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$*', d['value'], d['ms_per_step'], d['clocks']['sm_mhz'])"; }
( for i in 1 2; do
    b POETX_X=1
    b POETX_OUTER_SM_PCT=30
    b POETX_OUTER_SM_PCT=55
    b POETX_LIB_PATH=abtest/lib_bd51.so
  done ) > gpurun_out/tune.txt 2>&1
