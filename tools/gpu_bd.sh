mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_tc.py -x -q > gpurun_out/tc_tests.log 2>&1; echo "rc=$?" >> gpurun_out/tc_tests.log
timeout 300 python tools/microbench.py hbm > gpurun_out/mb_hbm.txt 2>&1
