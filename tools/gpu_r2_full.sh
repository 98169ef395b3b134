# full GPU suite + smoke + graph step breakdown
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke $?
timeout 1800 python -m pytest tests -q -m gpu --timeout 900 -rf > gpurun_out/gputest.log 2>&1; echo tests $?
timeout 600 python tools/profile_step.py --graph --timeline > gpurun_out/step_breakdown_graph.txt 2>&1; echo prof $?
tail -3 gpurun_out/smoke.log; tail -5 gpurun_out/gputest.log; head -22 gpurun_out/step_breakdown_graph.txt; grep -A12 "ONE kernel" gpurun_out/step_breakdown_graph.txt
