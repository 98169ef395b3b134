# same-box A/B of an environment toggle, alternating:
#   bash tools/gpu_envab.sh "POETX_X=0" [rounds] [extra bench.py args]
mkdir -p gpurun_out
alt=$1; n=${2:-3}; extra=${3:-}
( for i in $(seq $n); do
    for e in "$alt" "POETX_NOTHING=1"; do
      env $e timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-extras $extra | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$e', d['value'], d['ms_per_step'], d['clocks']['sm_mhz'])"
    done
  done
) >> gpurun_out/envab.txt 2>&1
cat gpurun_out/envab.txt
