# round-end evidence refresh: tests, smoke, bench (+reference arm), launch list, configs
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.log 2>&1
timeout 600 python bench.py --impl reference --steps 2 --warmup 0 > gpurun_out/bench_ref.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 4500 -c 2400 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-graph > gpurun_out/ncu_launch_bench.log 2>&1
timeout 600 python tools/profile_step.py --graph --timeline > gpurun_out/step_breakdown_graph.txt 2>&1
timeout 2400 python tools/configs_bench.py --out gpurun_out/configs.jsonl > gpurun_out/configs.log 2>&1
