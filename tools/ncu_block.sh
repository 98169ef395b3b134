mkdir -p gpurun_out
timeout 300 ncu --set full --clock-control none --import-source on -k regex:bd_kernel -s 2 -c 1 -o gpurun_out/bd_2048 python tools/blockbench.py apply 2048 > gpurun_out/ncu_bd.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:tc_kernel -s 2 -c 1 -o gpurun_out/outer_2048 python tools/blockbench.py outer 2048 > gpurun_out/ncu_outer.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:reduce_splits -s 2 -c 1 -o gpurun_out/reduce_2048 python tools/blockbench.py outer 2048 > gpurun_out/ncu_reduce.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:bd_kernel -s 2 -c 1 -o gpurun_out/bd_5632 python tools/blockbench.py apply 5632 > gpurun_out/ncu_bd2.log 2>&1
