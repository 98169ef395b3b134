mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_rowops.py tests/test_gpu_parity.py -x -q -k "permute or premerge or blockdiag or bf16" > gpurun_out/perm_tests.log 2>&1; echo "rc=$?" >> gpurun_out/perm_tests.log
timeout 300 python tools/microbench.py hbm 2>&1 | grep permute > gpurun_out/mb_perm.txt
POETX_PERMUTE_T8=0 timeout 300 python tools/microbench.py hbm 2>&1 | grep permute >> gpurun_out/mb_perm.txt
