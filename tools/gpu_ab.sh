# same-box A/B of two library builds: bash tools/gpu_ab.sh abtest/lib_prev.so [rounds]
mkdir -p gpurun_out
alt=$1; n=${2:-3}
( for i in $(seq $n); do
    for lib in "$alt" ""; do
      POETX_LIB_PATH=$lib timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('${lib:-current}', d['value'], d['ms_per_step'], d['clocks']['sm_mhz'])"
    done
  done
) > gpurun_out/ab.txt 2>&1
