mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_rowops.py -x -q > gpurun_out/rowops.log 2>&1
timeout 300 python tools/microbench.py rows > gpurun_out/mb_rows.txt 2>&1
POETX_ROWPIPE_RESIDENT=1 timeout 300 python tools/microbench.py rows > gpurun_out/mb_rows_res.txt 2>&1
