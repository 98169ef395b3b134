mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_tc.py -x -q -k "pair" > gpurun_out/pair_tests.log 2>&1
timeout 300 python tools/microbench.py gemm > gpurun_out/mb_gemm.txt 2>&1
