# 512-row pair tiles: tail 4 vs 3 -- microbench + step A/B
mkdir -p gpurun_out; rm -f gpurun_out/envab.txt
( echo "== tail 3"; timeout 300 python tools/microbench.py gemm
  echo "== tail 4"; POETX_LIB_PATH=abtest/lib_tail4.so timeout 300 python tools/microbench.py gemm ) > gpurun_out/microbench_tail4.txt 2>&1
POETX_LIB_PATH=abtest/lib_tail4.so timeout 1200 python -m pytest tests/test_gpu_tc.py tests/test_gpu_q8_gemm.py -x -q 2>&1 | tail -1 > gpurun_out/tail4_tests.txt
bash tools/gpu_envab.sh "POETX_LIB_PATH=abtest/lib_tail4.so" 3
cat gpurun_out/microbench_tail4.txt gpurun_out/tail4_tests.txt
