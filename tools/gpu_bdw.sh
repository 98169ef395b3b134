mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_tc.py -x -q -k blockdiag > gpurun_out/bd_tests.log 2>&1; echo "rc=$?" >> gpurun_out/bd_tests.log
timeout 300 python tools/microbench.py hbm 2>&1 | grep apply > gpurun_out/mb_bd.txt
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1
