mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests.log
timeout 300 python tools/microbench.py hbm > gpurun_out/mb_hbm.txt 2>&1
POETX_GEMM_PAIR=0 timeout 300 python tools/microbench.py hbm > gpurun_out/mb_hbm_1cta.txt 2>&1
timeout 300 python tools/microbench.py cnp > gpurun_out/mb_cnp.txt 2>&1
POETX_GEMM_PAIR=0 timeout 300 python tools/microbench.py cnp >> gpurun_out/mb_cnp.txt 2>&1
