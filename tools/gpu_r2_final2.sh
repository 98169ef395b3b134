# round-2 final evidence after the CNP rework: smoke, GPU suite, bench (+reference arm), launch list, step breakdown
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke $?
timeout 1800 python -m pytest tests -q -m gpu --timeout 900 -rf > gpurun_out/gputest.log 2>&1; echo tests $?
timeout 1200 python bench.py --steps 20 --warmup 3 > gpurun_out/bench_full.log 2>&1; echo bench $?
timeout 600 python bench.py --impl reference --steps 2 --warmup 0 > gpurun_out/bench_ref.log 2>&1; echo ref $?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 4500 -c 2400 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-graph --no-extras > gpurun_out/ncu_launch_bench.log 2>&1; echo ncu $?
timeout 600 python tools/profile_step.py --graph --timeline --steps 4 > gpurun_out/step_breakdown_graph.txt 2>&1; echo prof $?
tail -2 gpurun_out/smoke.log; tail -3 gpurun_out/gputest.log
grep '^{' gpurun_out/bench_full.log | python -c "
import json,sys; d=json.loads(sys.stdin.read())
for k in ['value','ms_per_step','e2e','roofline','step_tc_roofline','merge','mem_variant','xq_variant','lora_same_box','north_star_check','peak_hbm_gb','clocks','gpu_launches']: print(k, d.get(k))"
tail -1 gpurun_out/bench_ref.log | cut -c1-300
python tools/launch_summary.py gpurun_out/launches.csv | head -22
