mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_tc.py tests/test_gpu_trainer.py -x -q > gpurun_out/tc_tests.log 2>&1
timeout 300 python tools/microbench.py cnp > gpurun_out/mb_cnp.txt 2>&1
timeout 300 python tools/profile_step.py --rows 40 > gpurun_out/step_breakdown.txt 2>&1
