# round-2 evidence: GEMM traffic capture, bench launch list, step breakdown, full bench
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none -k regex:tc2_kernel -o gpurun_out/gemm_shapes python tools/gemm_shapes.py > gpurun_out/ncu_gemm_shapes.log 2>&1; echo ncu_shapes $?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 4500 -c 2400 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-graph --no-extras > gpurun_out/ncu_launch_bench.log 2>&1; echo ncu_launch $?
timeout 600 python tools/profile_step.py --graph --timeline > gpurun_out/step_breakdown_graph.txt 2>&1; echo prof $?
timeout 1200 python bench.py --steps 20 --warmup 3 > gpurun_out/bench_full.log 2>&1; echo bench $?
grep '^{' gpurun_out/bench_full.log | python -c "
import json,sys; d=json.loads(sys.stdin.read())
for k in ['value','ms_per_step','e2e','roofline','step_tc_roofline','merge','mem_variant','lora_same_box','north_star_check','peak_hbm_gb','clocks']: print(k, d.get(k))"
python tools/launch_summary.py gpurun_out/launches.csv | head -30
