# CNP launches in whole waves: trainer parity tests + same-box A/B (POETX_CNP_WAVES=0: one launch per decoder block)
mkdir -p gpurun_out; rm -f gpurun_out/envab.txt
timeout 1800 python -m pytest tests/test_gpu_bench_config.py tests/test_gpu_trainer.py tests/test_gpu_dp.py tests/test_gpu_cnp_fused.py -q -x 2>&1 | tail -2 > gpurun_out/waves_tests.txt
bash tools/gpu_envab.sh "POETX_CNP_WAVES=0" 3
bash tools/gpu_envab.sh "POETX_CNP_WAVES=0" 2 "--variant mem"
cat gpurun_out/waves_tests.txt
