mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_trainer.py -x -q > gpurun_out/trainer_tests.log 2>&1; echo "rc=$?" >> gpurun_out/trainer_tests.log
timeout 400 python tools/profile_step.py --graph > gpurun_out/step_breakdown_graph.txt 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1
