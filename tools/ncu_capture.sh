#!/bin/bash
# ncu evidence for profiles/: launch list of one bench step + full capture of the top kernel.
set -x
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 2500 -c 3000 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_kernel -s 300 -c 2 \
  -o gpurun_out/prof_tc python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:permute_cols_bf16 -s 100 -c 1 \
  -o gpurun_out/prof_perm python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_perm.log 2>&1
ls -la gpurun_out
