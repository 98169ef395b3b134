mkdir -p gpurun_out
( for c in 1b-poetxq-mem 1b-poetxq-mem 1b-poetx-mem 1b-poetxq-mem 8b-poetx-mem 8b-poetx-mem; do
    echo "$c: $(timeout 600 python tools/configs_bench.py --one $c 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(round(d.get('tokens_per_s',0)), round(d.get('ms_per_step',0),1), round(d.get('peak_hbm_gb',0),1))")"
  done
  nvidia-smi --query-gpu=clocks.sm,clocks_throttle_reasons.active,temperature.gpu,power.draw --format=csv
) > gpurun_out/ab_cfg.txt 2>&1
