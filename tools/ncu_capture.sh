#!/bin/bash
# ncu evidence for profiles/: per-kernel breakdown of one step (torch.profiler/CUPTI),
# the ncu launch list of a bench step, and full captures of the top kernels.
mkdir -p gpurun_out
timeout 600 python tools/profile_step.py --rows 60 > gpurun_out/step_breakdown.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 2500 -c 3000 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-graph > gpurun_out/ncu_launch_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_kernel -s 300 -c 2 \
  -o gpurun_out/prof_tc python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-graph > gpurun_out/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bd_kernel -s 100 -c 2 \
  -o gpurun_out/prof_bd python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-graph > gpurun_out/ncu_bd.log 2>&1
ls -la gpurun_out
