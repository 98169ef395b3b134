mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_trainer.py tests/test_gpu_bench_config.py tests/test_gpu_dp.py tests/test_checkpoint.py -q -m gpu -x -rf > gpurun_out/head_tests.log 2>&1; echo tests $?
tail -3 gpurun_out/head_tests.log
bash tools/gpu_envab.sh POETX_HEAD_SIDE=0 3
