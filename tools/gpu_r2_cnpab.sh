# step A/B of the CNP rework + CNP / trainer tests
mkdir -p gpurun_out; rm -f gpurun_out/envab.txt
timeout 1800 python -m pytest tests/test_gpu_cnp_fused.py tests/test_gpu_bench_config.py tests/test_gpu_parity.py tests/test_gpu_trainer.py tests/test_gpu_tc.py -q -x 2>&1 | tail -2 > gpurun_out/gputest_cnp.txt
bash tools/gpu_envab.sh "POETX_LIB_PATH=abtest/lib_cnp_old.so" 3
cat gpurun_out/gputest_cnp.txt
